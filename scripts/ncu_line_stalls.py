#!/usr/bin/env python3
"""Per-CUDA-line stall samples of an ncu capture (cuda,sass source view), for the
lines in [first, last]: samples share and the top two stall reasons.
usage: ncu_line_stalls.py report.ncu-rep first last [min_pct]"""
import csv
import io
import os
import subprocess
import sys

rep, lo, hi = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
minp = float(sys.argv[4]) if len(sys.argv) > 4 else 0.2
src = open(os.path.join(os.path.dirname(__file__), "..", "paper_1610_04124_b200", "csrc",
                        "kernels.cuh")).read().splitlines()
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
ix = {n: i for i, n in enumerate(hdr)}
cats = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]


def num(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


acc, cur, tot = {}, None, 0.0
for r in rows:
    if r and r[0].isdigit():
        cur = int(r[0])
        continue
    if len(r) < len(hdr) or not r[ix["Address"]].startswith("0x"):
        continue
    s = num(r[ix["Warp Stall Sampling (All Samples)"]])
    tot += s
    v = acc.setdefault(cur, [0.0] + [0.0] * len(cats))
    v[0] += s
    for k, c in enumerate(cats):
        v[k + 1] += num(r[ix[c]])
for ln in sorted(k for k in acc if k and lo <= k <= hi):
    v = acc[ln]
    if 100 * v[0] / tot < minp:
        continue
    top = sorted(zip(v[1:], cats), reverse=True)[:2]
    print(f"{ln:5d} {100 * v[0] / tot:5.2f}%  " + " ".join(f"{c[6:]}={100 * x / tot:.2f}" for x, c in top)
          + "  " + src[ln - 1].strip()[:60])
