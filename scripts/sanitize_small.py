#!/usr/bin/env python3
"""Small end-to-end run of the CUDA path for compute-sanitizer (memcheck /
racecheck / synccheck): a few columns of C1/C2-like frames in exact mode,
mean and median reductions (the row-wise register reduction on 16-byte aligned
frames, the tiled one otherwise), the f2 tables, D = 256, a dense-ring (wide
band) model and top-of-range pixels (L#27), each under both DP launch plans (4
and 8 warps per column); each result checked against the oracle."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from inputs import synth                                   # noqa: E402
from tests import modelparams as mp                        # noqa: E402
from tests.gpuharness import compare_exact, run_gpu, run_oracle   # noqa: E402

cases = []
sc = synth.c1_scene()
cases.append(("c1", mp.make(max_disparity=32, ground_slope=sc.alpha),
              np.stack([synth.render(sc, 1)])))
H, W, D = 100, 40, 64
fr = np.stack([synth.render(synth.random_scene(7, W, H, D, alpha=0.5), 7)])
cases.append(("rand", mp.make(max_disparity=D, ground_slope=0.5), fr))
cases.append(("median", mp.make(max_disparity=D, ground_slope=0.5, reduce_mode=1), fr))
cases.append(("dense", mp.make(max_disparity=D, ground_slope=0.5, sigma=(2.0, 3.0, 0.5)), fr))
rng = np.random.default_rng(1)
cases.append(("f2", mp.make(max_disparity=D, ground_slope=0.5,
                            sigma_object_f=rng.uniform(0.7, 2.0, D).astype(np.float32),
                            sigma_ground_v=rng.uniform(0.8, 3.0, H).astype(np.float32)), fr))
cases.append(("d256", mp.make(max_disparity=256, ground_slope=1.5),
              np.stack([synth.uniform_random_image(3, 30, 70, 256)])))
ft = rng.integers(62 << 4, 64 << 4, size=(1, 48, 1024)).astype(np.uint16)   # top of range, tight rows
cases.append(("top", mp.make(max_disparity=64, ground_slope=0.6), ft))
cases.append(("ragged", mp.make(max_disparity=D, ground_slope=0.5), np.ascontiguousarray(fr[:, :, :37])))
bad = 0
for name, p, frames in cases:
    o, oc = run_oracle(p, frames)
    for plan in (4, 8):
        g, gc, _, hd = run_gpu(p, frames, plan=plan)
        nb = len(compare_exact(g, gc, o, oc, p["cost_frac_bits"]))
        bad += nb
        print(f"{name} (plan {plan}): {len(g[0])} columns, mismatches {nb}")
sys.exit(1 if bad else 0)
