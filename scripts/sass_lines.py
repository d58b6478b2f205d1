#!/usr/bin/env python3
"""Static SASS size of one kernel per CUDA source line (instruction-cache
footprint): nvdisasm -g of the library's cubin.  usage: sass_lines.py
<kernel-mangled-substring> [top] [lib]"""
import os
import re
import subprocess
import sys
import tempfile

pat = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
lib = sys.argv[3] if len(sys.argv) > 3 else "paper_1610_04124_b200/libstixels.so"
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
cnt, cur, inside = {}, None, False
for line in dis.splitlines():
    if line.startswith("//----") and ".text." in line:
        inside = pat in line
        continue
    if not inside:
        continue
    m = re.search(r'//## File "([^"]+)", line (\d+)', line)
    if m:
        cur = (os.path.basename(m.group(1)), int(m.group(2)))
    elif re.match(r"\s+/\*[0-9a-f]{4,}\*/", line) and cur:
        cnt[cur] = cnt.get(cur, 0) + 1
srcs = {}
tot = sum(cnt.values())
print(f"{tot} instructions")
for (f, l), v in sorted(cnt.items(), key=lambda x: -x[1])[:top]:
    if f not in srcs:
        path = os.path.join("paper_1610_04124_b200", "csrc", f)
        srcs[f] = open(path).read().splitlines() if os.path.exists(path) else []
    txt = srcs[f][l - 1].strip()[:78] if l <= len(srcs[f]) else ""
    print(f"{v:5d} {f}:{l:<5d} {txt}")
