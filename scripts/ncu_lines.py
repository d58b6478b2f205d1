#!/usr/bin/env python3
"""Per-CUDA-source-line totals of an ncu report (needs -lineinfo): warp-instructions
executed and stall samples, top N lines.  usage: ncu_lines.py report [N] [ncols]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ncols = float(sys.argv[3]) if len(sys.argv) > 3 else 1.0
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[2]
data = rows[3:]
iline, isrc = 0, 1
iex = hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
acc = {}
for r in data:
    # line-level rows carry the line's aggregated metrics; SASS rows have an empty line
    if len(r) <= iex or not r[0].isdigit():
        continue
    key = (int(r[0]), r[1])
    a = acc.setdefault(key, [0, 0])
    try:
        a[0] += int(float(r[iex] or 0))
        a[1] += int(float(r[iss] or 0))
    except ValueError:
        pass
tot_i = sum(v[0] for v in acc.values())
tot_s = sum(v[1] for v in acc.values())
print(f"total instr {tot_i:,}  per column {tot_i / ncols:,.0f}")
for (ln, src), (ins, smp) in sorted(acc.items(), key=lambda kv: -kv[1][0])[:N]:
    print(f"{ln:5d} {100 * ins / tot_i:5.1f}% {ins / ncols:9.0f}/col  samp {100 * smp / max(tot_s, 1):5.1f}%  {src.strip()[:70]}")
