#!/usr/bin/env python3
"""Phase timeline of dp_kernel's third column per column group of CTA 0 (diagnostic
build libstixels_trace.so, -DSTX_TRACE).  Prints, per 32-row block b, cycles
relative to the block start: serial triangle done, build done, each warp's bulk
end, the bar release, each warp's newest-chunk end, the block end.
usage (GPU box): python scripts/trace_phases.py [batch] [warps_per_column]"""
import ctypes
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1610_04124_b200 import build as B          # noqa: E402
from paper_1610_04124_b200 import stixels as S        # noqa: E402
from inputs import synth                              # noqa: E402
from tests import modelparams as mp                   # noqa: E402

lib = ctypes.CDLL(B.build(trace=True))
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
W, H = 1024, 440
p = S.params_from_dict(mp.make(), H)
h = ctypes.c_void_p()
assert lib.stixels_create(ctypes.byref(p), W, H, batch, 0, None, ctypes.byref(h)) == 0
pool = np.stack([synth.frame(3, i, W, H, 128) for i in range(16)])
disp = torch.from_numpy(pool.view(np.int16)).cuda()[torch.arange(batch) % 16]
nc = W // 5
out = torch.empty((batch, nc, H, 12), dtype=torch.uint8, device="cuda")
cnt = torch.empty((batch, nc), dtype=torch.int32, device="cuda")
tr = torch.zeros(4 * 64 * 32, dtype=torch.int64, device="cuda")
lib.stixels_trace_buffer(h, ctypes.c_void_p(tr.data_ptr()))
P = lambda t: ctypes.c_void_p(t.data_ptr())
cw = int(sys.argv[2]) if len(sys.argv) > 2 else 0
if cw:
    assert lib.stixels_set_launch_plan(h, cw) == 0
for _ in range(2):
    assert lib.stixels_compute(h, P(disp), ctypes.c_int64(W * 2), batch, P(out), P(cnt), None) == 0
torch.cuda.synchronize()
t = tr.cpu().numpy().reshape(4, 64, 32).astype(np.int64)
t = t * 1.965          # globaltimer ns -> cycles at 1965 MHz
nb = (H + 31) // 32
names = ["setup", "chain", "scans", "tri", "build"] + [f"bulk{i}" for i in range(8)] + ["rel"] + \
        [f"new{i}" for i in range(8)] + ["end"]
slots = [21, 22, 23, 1, 2] + list(range(3, 11)) + [11] + list(range(12, 20)) + [20]
for g in range(4):
    print(f"group {g}: block start-to-start ~cycles (globaltimer ns x 1.965) and phase ends (relative to block start)")
    print("  b  " + " ".join(f"{n:>6s}" for n in names))
    tot = 0
    for b in range(nb):
        r = t[g, b]
        if r[0] == 0:
            continue
        rel = [(int(r[s] - r[0]) if r[s] else -1) for s in slots]
        tot += rel[-1]
        print(f" {b:2d}  " + " ".join(f"{x:6d}" for x in rel))
    print(f"  column total {tot} cycles")
    it = t[g, 60]
    if it[0]:
        b0 = t[g, 0, 0]
        print(f"  item start -> block 0 start {int(b0 - it[0])} (prologue A {int(it[3] - it[0])}, "
              f"B {int(it[4] - it[3])}, build {int(it[5] - it[4])}, block-0 cells {int(b0 - it[5])}), "
              f"blocks {int(it[1] - b0)}, backtrack+write {int(it[2] - it[1])} cycles")
