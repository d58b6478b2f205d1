#!/usr/bin/env python3
"""Frames/s of the whole path at one shape (A/B helper).
usage: time_shape.py W H [s] [D] [batch] [lib.so]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1610_04124_b200 import stixels as S   # noqa: E402
from inputs import synth                          # noqa: E402
from tests import modelparams as mp               # noqa: E402

W, H = int(sys.argv[1]), int(sys.argv[2])
s = int(sys.argv[3]) if len(sys.argv) > 3 else 5
D = int(sys.argv[4]) if len(sys.argv) > 4 else 128
B = int(sys.argv[5]) if len(sys.argv) > 5 else 1024
if len(sys.argv) > 6:
    S.use_library(sys.argv[6])
p = mp.make(max_disparity=D, stixel_width=s)
pool = np.stack([synth.frame(4, i, W, H, D) for i in range(8)])
disp = torch.from_numpy(pool.view(np.int16)).cuda()[torch.arange(B) % 8]
hd = S.Handle(S.params_from_dict(p, H), W, H, B)
out, cnt, cost = hd.alloc_outputs(B)
for _ in range(2):
    hd.compute(disp, out, cnt, cost)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(3):
    hd.compute(disp, out, cnt, cost)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 3
print(f"{W}x{H} s={s} D={D} B={B}: {B / ms * 1000:.0f} frames/s ({ms:.2f} ms)")
