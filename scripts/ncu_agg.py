#!/usr/bin/env python3
"""Aggregate stall samples of an ncu report over SASS offset ranges.
usage: ncu_agg.py report name:lo-hi [name:lo-hi ...]"""
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
ia, iss, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
isel = hdr.index("stall_selected")
base = int(data[0][ia], 16)
tot = sum(int(r[iss]) for r in data)
agg = {}
for r in data:
    off = int(r[ia], 16) - base
    name = "other"
    for n, lo, hi in ranges:
        if lo <= off <= hi:
            name = n
            break
    a = agg.setdefault(name, [0, 0, 0])
    a[0] += int(r[iss]); a[1] += int(r[iex]); a[2] += int(r[isel] or 0)
for n, (s, e, sel) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{n:14s} samples {100*s/tot:5.1f}%  issued {100*sel/max(s,1):5.1f}% of its samples  instr {e:13d}")
