#!/usr/bin/env python3
"""List the loops (backward branches) of a kernel in libstixels.so with their
instruction / LDS / STS counts.  Usage: sass_loops.py <kernel-substring> [max_len]"""
import re
import subprocess
import sys

lib = sys.argv[3] if len(sys.argv) > 3 else "paper_1610_04124_b200/libstixels.so"
pat = sys.argv[1] if len(sys.argv) > 1 else "dp_kernelILi128"
maxlen = int(sys.argv[2]) if len(sys.argv) > 2 else 400
txt = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
for f in re.split(r"\n\s+Function : ", txt)[1:]:
    name = f.split("\n")[0]
    if pat not in name:
        continue
    ins = []
    for line in f.splitlines():
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    open("/tmp/kernel.sass", "w").write("\n".join(f"{a:05x} {t}" for a, t in ins))
    print(name, len(ins), "instructions")
    for a, t in ins:
        m = re.search(r"BRA (0x[0-9a-f]+)", t)
        if m and "DIV" not in t:
            tgt = int(m.group(1), 16)
            if tgt < a:
                body = [x for x in ins if tgt <= x[0] <= a]
                if len(body) <= maxlen:
                    c = lambda s: sum(s in x[1] for x in body)
                    print(f"  loop {tgt:#06x}-{a:#06x}: {len(body)} instr, LDS {c('LDS')}, STS {c('STS')}, "
                          f"SHFL {c('SHFL')}, FADD {c('FADD')}, SEL {c('SEL')}, SETP {c('SETP')}")
