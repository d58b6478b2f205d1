#!/usr/bin/env python3
"""Per-phase totals of a dp_kernel ncu capture (needs -lineinfo): warp-instructions,
shared-memory wavefronts and stall samples per column, with the phases located by
marker lines of kernels.cuh.  usage: ncu_phases.py report.ncu-rep [n_columns]"""
import csv
import io
import os
import subprocess
import sys

rep = sys.argv[1]
ncol = float(sys.argv[2]) if len(sys.argv) > 2 else 52224.0
src = open(os.path.join(os.path.dirname(__file__), "..", "paper_1610_04124_b200", "csrc", "kernels.cuh")).read().splitlines()
marks = [("auto rect_run", "rect_run"), ("auto merge_part", "merge_part"), ("auto bulk_chunks", "bulk_chunks"),
         ("prologue A", "prologue"), ("auto build_priv", "build_priv"), ("auto precompute_cells", "precompute"),
         ("auto copy_seed", "copy_seed"), ("block 0 has only", "block0"), ("for (int b = 0; b < nb; ++b)", "block-serial"),
         ("for (int jp = 0; jp < jn; ++jp)", "chain"), ("STX_STAMP(b, 22)", "block-serial"),
         ("all warps: block b+1", "block-rect"), ("backtracking (P:159)", "backtrack")]
starts = []
for i, l in enumerate(src, 1):
    for m, n in marks:
        if m in l:
            starts.append((i, n))
            break
starts.sort()
kbeg = next(i for i, l in enumerate(src, 1) if "__global__ void __launch_bounds__(32 * kCW" in l)


def phase(ln):
    if ln < kbeg:
        return "helpers"
    cur = "kernel-setup"
    for i, n in starts:
        if i <= ln:
            cur = n
    return cur


raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))


def num(x):
    try:
        return int(float(x))
    except ValueError:
        return 0


acc, cur = {}, "?"
for r in rows[3:]:
    if r and r[0].isdigit():
        cur = phase(int(r[0]))
        continue
    if len(r) < 22 or not r[2].startswith("0x"):
        continue
    v = acc.setdefault(cur, [0, 0, 0, 0])
    v[0] += num(r[7]); v[1] += num(r[19]); v[2] += num(r[18]); v[3] += num(r[4])
ts = sum(v[3] for v in acc.values())
ti = sum(v[0] for v in acc.values())
tw = sum(v[1] for v in acc.values())
print(f"{'phase':14s} {'instr/col':>10s} {'wf/col':>8s} {'excess':>7s} {'samples':>8s}")
for k, v in sorted(acc.items(), key=lambda kv: -kv[1][0]):
    print(f"{k:14s} {v[0]/ncol:10.0f} {v[1]/ncol:8.0f} {v[2]/ncol:7.0f} {100*v[3]/ts:7.1f}%")
print(f"{'total':14s} {ti/ncol:10.0f} {tw/ncol:8.0f}")
