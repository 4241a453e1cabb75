#!/usr/bin/env python3
"""Text summary of an `ncu --set full` report (one block per captured kernel):
duration, DRAM bytes, fp64 tensor-pipe activity, warps active, top stall reasons.

    python tools/ncu_summary.py gpurun_out/prof_chol_xl_r02a.ncu-rep [label] > profiles/ncu_....txt
Prints one trailing JSON line {"dram_bytes_per_launch": [...]} for profiles/ncu_traffic.json.
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration", "us"),
    ("launch__grid_size", "grid", ""),
    ("launch__block_size", "block", ""),
    ("launch__registers_per_thread", "registers/thread", ""),
    ("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "DMMA pipe active (% of active cycles)", "%"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active (% of elapsed)", "%"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active (% of 64/SM)", "%"),
    ("dram__bytes_read.sum", "DRAM read", "MB"),
    ("dram__bytes_write.sum", "DRAM write", "MB"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate", "%"),
    ("smsp__inst_executed.sum", "warp instructions", ""),
]


def main():
    rep = sys.argv[1]
    label = sys.argv[2] if len(sys.argv) > 2 else rep
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    print(f"# ncu --set full --clock-control none: {label}")
    print(f"# report: {rep}")
    traffic = []
    for r in data:
        print(f"\n== {r[col['Kernel Name']][:110]}")
        for key, name, unit in METRICS:
            if key not in col:
                continue
            v = r[col[key]]
            u = units[col[key]]
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                print(f"  {name}: {v}")
                continue
            if key.startswith("dram__bytes"):
                x = x * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
                print(f"  {name}: {x:.1f} MB")
            elif key == "gpu__time_duration.sum":
                x = x * {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}.get(u, 1.0)
                print(f"  {name}: {x:.1f} us")
            else:
                print(f"  {name}: {x:g}{unit if unit not in ('', 'MB') else ''}")
        rd = float(r[col["dram__bytes_read.sum"]].replace(",", ""))
        wr = float(r[col["dram__bytes_write.sum"]].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(units[col["dram__bytes_read.sum"]], 1)
        traffic.append(int((rd + wr) * scale))
        st = {h[33:]: float(r[i] or 0) for h, i in col.items()
              if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued")}
        tot = sum(st.values()) or 1.0
        top = sorted(st.items(), key=lambda t: -t[1])[:7]
        print("  warp stall samples: " + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
    print(json.dumps({"dram_bytes_per_launch": traffic}))


if __name__ == "__main__":
    main()
