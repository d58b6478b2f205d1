#!/usr/bin/env python3
"""Stall-reason breakdown (share of samples) per SASS offset range of an ncu report.
usage: ncu_stalls.py report name:lo-hi [name:lo-hi ...]   (first matching range wins)"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ranges = []
for spec in sys.argv[2:]:
    n, r = spec.split(":")
    lo, hi = r.split("-")
    ranges.append((n, int(lo, 16), int(hi, 16)))
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
ia, iss = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
tot = sum(int(r[iss]) for r in data)
agg = {}
for r in data:
    off = int(r[ia], 16) - base
    name = next((n for n, lo, hi in ranges if lo <= off <= hi), "other")
    a = agg.setdefault(name, [0] * (len(sc) + 1))
    a[0] += int(r[iss])
    for q, i in enumerate(sc):
        a[q + 1] += int(float(r[i] or 0))
for n, a in sorted(agg.items(), key=lambda x: -x[1][0]):
    parts = sorted(((a[q + 1], hdr[i][6:]) for q, i in enumerate(sc)), reverse=True)[:7]
    print(f"{n:8s} {100*a[0]/tot:5.1f}%  " + "  ".join(f"{k}={100*v/max(a[0],1):.0f}%" for v, k in parts))
