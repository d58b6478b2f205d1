#!/usr/bin/env python3
"""Shared-memory instructions with the most excess (bank-conflict) wavefronts.
usage: ncu_conflicts.py report.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
ia, isrc = hdr.index("Address"), hdr.index("Source")
iw, ii, iex = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal"), hdr.index("Instructions Executed")
base = int(data[0][ia], 16)
num = lambda s: int(float(s or 0))
tw = sum(num(r[iw]) for r in data); ti = sum(num(r[ii]) for r in data)
print(f"wavefronts {tw:,}  ideal {ti:,}  excess {tw - ti:,}")
for r in sorted(data, key=lambda r: -(num(r[iw]) - num(r[ii])))[:N]:
    w, i = num(r[iw]), num(r[ii])
    print(f"{int(r[ia],16)-base:#07x} excess={w-i:12,d} wf={w:12,d} ex={num(r[iex]):11,d}  {r[isrc][:60]}")
