#!/usr/bin/env python3
"""Per-instruction stall samples of an ncu report, top-N, with SASS offsets.
usage: ncu_regions.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iss, iex = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
tot = sum(int(r[iss]) for r in data)
print("total samples", tot)
for r in sorted(data, key=lambda r: -int(r[iss]))[:N]:
    print(f"{int(r[ia],16)-base:#07x} {int(r[iss]):8d} {100*int(r[iss])/tot:5.1f}% ex={int(r[iex]):11d}  {r[isrc][:60]}")
