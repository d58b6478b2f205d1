#!/usr/bin/env python3
"""Stall reasons per instruction in a SASS offset range of an ncu report.
usage: ncu_range.py report.ncu-rep lo hi"""
import csv
import io
import subprocess
import sys

rep, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
agg = {r: 0 for r in reasons}
tot = 0
for r in data:
    off = int(r[ia], 16) - base
    if lo <= off <= hi:
        s = int(r[iss]); tot += s
        top = sorted(((int(r[hdr.index(x)] or 0), x[6:]) for x in reasons), reverse=True)[:3]
        for x in reasons:
            agg[x] += int(r[hdr.index(x)] or 0)
        print(f"{off:#07x} {s:7d} {r[isrc][:48]:48s} " + " ".join(f"{n}={v}" for v, n in top if v))
print("range total", tot, {k[6:]: v for k, v in sorted(agg.items(), key=lambda x: -x[1]) if v})
