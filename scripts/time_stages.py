#!/usr/bin/env python3
"""Single-frame stage latency (GPU box): CUDA-event time per call of
stixels_reduce, stixels_solve and stixels_compute on one 1024x440 frame, for
each DP launch plan.  usage: python scripts/time_stages.py [frames_per_call]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1610_04124_b200 import stixels as S   # noqa: E402
from inputs import synth                         # noqa: E402
from tests import modelparams as mp              # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
libs = sys.argv[2:] or [None]
W, H = 1024, 440
pool = np.stack([synth.frame(2, i, W, H, 128) for i in range(8)])
disp = torch.from_numpy(pool.view(np.int16)).cuda()
import ctypes
for lib in libs:
  S._lib = None
  S.use_library(lib or S.LIB) if lib else None
  for plan in ((0, 4, 8) if lib is None else (8,)):
      hd = S.Handle(S.params_from_dict(mp.make(), H), W, H, B)
      hd.set_launch_plan(plan)
      out, cnt, cost = hd.alloc_outputs(B)
      cols = torch.empty((B, hd.n_cols, H), dtype=torch.int16, device="cuda")
      res = {}
      for name in ("reduce", "solve", "compute"):
          def call(i):
              x = disp[(i * B) % 8:(i * B) % 8 + B] if B <= 8 else disp[torch.arange(B) % 8]
              if name == "reduce":
                  hd.reduce(x, cols)
              elif name == "solve":
                  hd.solve(cols, out, cnt, cost)
              else:
                  hd.compute(x, out, cnt, cost)
          for i in range(5):
              call(i)
          torch.cuda.synchronize()
          e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
          n = 40
          e0.record()
          for i in range(n):
              call(i)
          e1.record()
          torch.cuda.synchronize()
          res[name] = 1000.0 * e0.elapsed_time(e1) / n
      print(f"{os.path.basename(lib or 'product')} plan {plan} (ran {hd.last_launch_shape()}): " +
            ", ".join(f"{k} {v:.1f} us" for k, v in res.items()))
      hd.destroy()
