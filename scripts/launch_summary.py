#!/usr/bin/env python3
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel totals and shares.  usage: launch_summary.py launches.csv [title]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr, data = rows[hi], rows[hi + 1:]
ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
tot = {}
for r in data:
    if len(r) <= iv:
        continue
    name = r[ik].split("(")[0]
    tot.setdefault(name, []).append(float(r[iv].replace(",", "")) * scale[r[iu]])
allt = sum(sum(v) for v in tot.values())
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print("(cold-cache, serialised launches under ncu: compare shares, not absolute times)")
for k, v in sorted(tot.items(), key=lambda x: -sum(x[1])):
    print(f"{k:40s} launches {len(v):3d}  total {sum(v):9.3f} ms  mean {sum(v)/len(v):8.3f} ms  share {100*sum(v)/allt:6.2f}%")
