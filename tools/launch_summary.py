#!/usr/bin/env python3
"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (last run only)."""
import collections
import csv
import sys


def main(fn, runs=2):
    rows = list(csv.reader(open(fn)))
    hdr_i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[hdr_i], rows[hdr_i + 1:]
    ki, vi, mi = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
    recs = [(r[ki], float(r[vi])) for r in data if r[mi] == "gpu__time_duration.sum"]
    # drop setup kernels (before the first schedule kernel), keep the last run
    recs = [r for r in recs if "spd_product" not in r[0]]
    per = len(recs) // runs
    last = recs[-per:] if per else recs
    agg = collections.defaultdict(lambda: [0, 0.0])
    for k, v in last:
        short = k.split("(")[0].replace("void ", "").split("::")[-1][:48]
        agg[short][0] += 1
        agg[short][1] += v
    tot = sum(v for _, v in last)
    print(f"{fn}: {len(last)} kernels, serialized sum {tot / 1e3:.1f} us")
    for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1])[:10]:
        print(f"  {k:48s} n={c:4d} total={v / 1e3:8.1f}us avg={v / c / 1e3:7.2f}us share={v / tot:.2f}")


if __name__ == "__main__":
    for f in sys.argv[1:]:
        main(f)
