"""Helpers running the same seeded frames through the CUDA path (C ABI) and the
oracle, and comparing them.  Imported by GPU tests, smoke() and bench.py."""
from __future__ import annotations

import numpy as np

from tests import modelparams as mp


def run_gpu(p: dict, frames: np.ndarray, max_batch: int | None = None, host: bool = False,
            plan: int = 0, bound: int = 0):
    """frames: [B][H][W] uint16/uint8/float32 -> (lists per frame per column, costs [B][n_cols],
    counts [B][n_cols], handle).  plan: DP launch plan (0 auto, 4 or 8 warps per column;
    a forced plan is checked against the launch the library reports; bound: the int32
    kernel's chunk bound, 0 auto, 1 off, 2 on)."""
    import torch
    from paper_1610_04124_b200 import stixels as S
    B, H, W = frames.shape
    params = S.params_from_dict(p, H)
    if frames.dtype == np.uint8:
        params.disp_format = S.U8
    elif frames.dtype == np.float32:
        params.disp_format = S.F32
    hd = S.Handle(params, W, H, max_batch or B)
    if plan:
        hd.set_launch_plan(plan)
    if bound:
        hd.set_chunk_bound(bound)
    if host:
        out = np.zeros((B, hd.n_cols, hd.cap, 12), np.uint8)
        cnt = np.zeros((B, hd.n_cols), np.int32)
        cost = np.zeros((B, hd.n_cols), np.float32)
        hd.compute_host(np.ascontiguousarray(frames), out, cnt, cost)
    else:
        t = torch.from_numpy(np.ascontiguousarray(frames).view(np.int16) if frames.dtype == np.uint16
                             else np.ascontiguousarray(frames)).cuda()
        out, cnt, cost = hd.alloc_outputs(B)
        hd.compute(t, out, cnt, cost)
        hd.sync()
        out, cnt, cost = out.cpu().numpy(), cnt.cpu().numpy(), cost.cpu().numpy()
    if plan:
        assert hd.last_launch_shape()[0] == plan, hd.last_launch_shape()
    return S.decode(out, cnt), cost, cnt, hd


def run_oracle(p: dict, frames: np.ndarray, cols_subset=None, threads: int = 0):
    """Oracle on every (or a subset of) column(s) of every frame."""
    from oracle import oracle as orc
    B, H, W = frames.shape
    m = mp.oracle_model(p, H)
    res, costs = [], []
    for b in range(B):
        cols = orc.reduce(frames[b], p["stixel_width"], p["disp_frac_bits"],
                          p["invalid_value"], p["max_disparity"], mode=p.get("reduce_mode", 0))
        if cols_subset is not None:
            cols = cols[cols_subset[b]]
        st, c = orc.solve_frame(m, cols, mode=1, threads=threads)
        res.append(st)
        costs.append(c)
    return res, costs


def compare_exact(gpu_lists, gpu_cost, ora_lists, ora_cost, scale_q: int):
    """Exact mode: identical lists (classes, bounds, disparities) and identical
    column costs (both are the same integer number of 2^-q quanta)."""
    bad = []
    for b in range(len(ora_lists)):
        for c in range(len(ora_lists[b])):
            o = [(vb, vt, cl, float(np.float32(d))) for vb, vt, cl, d in ora_lists[b][c]]
            g = gpu_lists[b][c]
            oc = np.float32(ora_cost[b][c] * 2.0 ** -scale_q) if scale_q else np.float32(ora_cost[b][c])
            gc = np.float32(gpu_cost[b][c])
            if o != g or oc != gc:
                bad.append((b, c, o, g, float(oc), float(gc)))
    return bad
