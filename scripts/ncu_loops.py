#!/usr/bin/env python3
"""Per-loop breakdown of an ncu report: samples, issue fraction, instructions and
shared wavefronts per column, using the loops of the current libstixels.so SASS.
usage: ncu_loops.py report kernel_substring n_columns"""
import csv
import io
import re
import subprocess
import sys

rep, pat, ncol = sys.argv[1], sys.argv[2], float(sys.argv[3])
loops_txt = subprocess.run([sys.executable, "scripts/sass_loops.py", pat, "100000"],
                           capture_output=True, text=True).stdout
loops = []
for l in loops_txt.splitlines():
    m = re.search(r"loop 0x([0-9a-f]+)-0x([0-9a-f]+): (\d+) instr", l)
    if m and int(m.group(3)) > 20:
        loops.append((int(m.group(1), 16), int(m.group(2), 16), int(m.group(3))))
# innermost first: sort by size
loops.sort(key=lambda x: x[1] - x[0])
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, data = rows[1], rows[2:]
ia, iss, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
isel, iwf = hdr.index("stall_selected"), hdr.index("L1 Wavefronts Shared")
ibar = hdr.index("stall_barrier")
base = int(data[0][ia], 16)
tot = sum(int(r[iss]) for r in data)
agg = {}
for r in data:
    off = int(r[ia], 16) - base
    key = "other"
    for a, b, n in loops:
        if a <= off <= b:
            key = f"{a:#06x}-{b:#06x}({n})"
            break
    s = agg.setdefault(key, [0, 0, 0, 0, 0])
    s[0] += int(r[iss]); s[1] += int(r[iex]); s[2] += int(r[isel] or 0); s[3] += int(r[iwf] or 0)
    s[4] += int(r[ibar] or 0)
print(f"{'region':24s} {'samples':>8s} {'barrier':>8s} {'issue%':>7s} {'instr/col':>10s} {'wf/col':>8s}")
for k, (s, e, sel, wf, br) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{k:24s} {100*s/tot:7.1f}% {100*br/tot:7.1f}% {100*sel/max(s,1):6.1f}% {e/ncol:10.0f} {wf/ncol:8.0f}")
