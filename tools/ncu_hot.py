#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from `ncu --page source --csv`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
# keep the first kernel section only (a CSV may hold several)
ends = [i for i, r in enumerate(rows) if i > 0 and r and r[0] == "Kernel Name"]
rows = rows[:ends[0]] if ends else rows
hdr = rows[1]
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
data = [r for r in rows[2:] if len(r) > si and r[si] not in ("", "0")]
tot = sum(float(r[si]) for r in data)
agg = {}
for r in data:
    for i in stall_cols:
        if r[i] not in ("", "0"):
            agg[hdr[i]] = agg.get(hdr[i], 0) + float(r[i])
print("total samples", tot)
print("stalls:", ", ".join(f"{k}={v / tot:.2f}" for k, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
for r in sorted(data, key=lambda r: -float(r[si]))[:n]:
    top = max(stall_cols, key=lambda i: float(r[i] or 0))
    print(f"{r[0][-5:]} {float(r[si]) / tot:5.3f} {hdr[top][6:]:>16s} {r[1].strip()[:90]}")
