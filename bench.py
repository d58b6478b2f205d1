#!/usr/bin/env python
"""Benchmark of the stixel hot path (BASELINE.json metric: frames/s at
1024x440 w=5 on 1/2/4/8 B200; DP cell-updates/s vs pipe peak).

One step = one pass of the whole hot path (reduction + DP + backtracking,
SURVEY 8(a) a1-a7) over one batch of synthetic frames resident in HBM:
config C3, 4096 frames of 1024x440, w=5, D=128 per rank.  Frames are
independent, so N ranks each process their own batch (weak scaling, no
collective on the data path; NCCL only carries the barrier and the max-over-
ranks timing).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the
reference arm for this paper-only tier) on the host cores.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/s at 1024x440 w=5 (1/2/4/8 B200); DP cell-updates/s vs pipe peak"
W_IMG, H_IMG, S_W, D_MAX = 1024, 440, 5, 128
ALG_OPS_PER_CELL = 20          # algorithmic work per DP cell


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=4096, help="frames per rank per step")
    ap.add_argument("--distinct", type=int, default=128, help="distinct seeded frames in the pool")
    ap.add_argument("--e2e-batch", type=int, default=1024)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-single", action="store_true", help="skip the one-frame latency run")
    ap.add_argument("--cpu-frames", type=int, default=0, help="oracle sample size (0 = auto)")
    ap.add_argument("--sweep", action="store_true",
                    help="NEXT f1: resolution / stixel-width sweep with fps/W (one JSON line "
                         "per config; not the driver's bench line)")
    ap.add_argument("--sweep-out", default="", help="also write the sweep lines to this file")
    ap.add_argument("--quality", type=int, default=0,
                    help="NEXT f3: Table-1 metrics (detection rate, false positives) of the "
                         "CUDA path on N noisy C2 frames against their synthetic ground truth")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def params_dict():
    from tests import modelparams as mp
    return mp.make()


def frame_indices(rank, n):
    """Seeded frame indices of a rank's pool (config 3 = C3): disjoint per rank,
    since frames are sharded (weak scaling, each rank owns its own batch)."""
    return [rank * 100000 + i for i in range(n)]


def frame_pool(n, rank):
    from inputs import synth
    return np.stack([synth.frame(3, i, W_IMG, H_IMG, D_MAX) for i in frame_indices(rank, n)])


def max_over_ranks(value, world, device=None):
    """Max of a per-rank time over all ranks (the job ends when the slowest rank
    does); a no-op at world size 1."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(frames_per_rank, steps, world, max_ms):
    """Whole-job throughput: frames of all ranks / slowest rank's time."""
    return frames_per_rank * world * steps / (max_ms / 1000.0)


def cells_per_frame():
    n_cols = W_IMG // S_W
    return n_cols * H_IMG * (H_IMG + 1) // 2


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()
        num = lambda x: x.replace(".", "").isdigit()
        sm = [float(r[0]) for r in self.rows if num(r[0])]
        mx = [float(r[1]) for r in self.rows if num(r[1])]
        pw = [float(r[2]) for r in self.rows if num(r[2])]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "power_w": statistics.median(pw) if pw else None, "samples": len(self.rows)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


def ncu_profile():
    """The committed ncu --set full capture of the DP kernel (profiles/): DRAM bytes
    per frame and measured pipe utilisations, or {}."""
    try:
        return json.load(open(os.path.join(ROOT, "profiles", "dp_kernel_ncu.json")))
    except Exception:
        return {}


def cpu_baseline(p, pool, frames_req=0):
    """The oracle (prefix mode, OpenMP over columns, all host cores) on a bounded
    sample of the same workload."""
    from tests.gpuharness import run_oracle
    from oracle import oracle as orc
    threads = orc.max_threads()
    n = frames_req or 1
    t0 = time.perf_counter()
    run_oracle(p, pool[:n], threads=threads)
    dt = time.perf_counter() - t0
    if not frames_req:
        # grow the sample to ~12 s of CPU work (the pool's frames repeat if needed)
        n = int(max(1, min(8 * len(pool), 12.0 / max(dt, 1e-3))))
        t0 = time.perf_counter()
        run_oracle(p, pool[np.arange(n) % len(pool)], threads=threads)
        dt = time.perf_counter() - t0
    return {"value": n / dt, "unit": "frames/s", "cores": threads, "kind": "oracle",
            "sample": f"{n} frames of C3 (1024x440, w=5, D=128{'; the pool of ' + str(len(pool)) + ' repeated' if n > len(pool) else ''}), oracle prefix mode O(h^2), "
                      f"double precision, OpenMP over columns, {threads} threads, {dt:.1f} s"}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands (the reference arm of a
    paper-only tier), on the host cores, same metric/config/unit."""
    if rank != 0:
        return
    p = params_dict()
    pool = frame_pool(4, 0)
    from tests.gpuharness import run_oracle
    from oracle import oracle as orc
    threads = orc.max_threads()
    per_step = 2
    for _ in range(args.warmup):
        run_oracle(p, pool[:per_step], threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        run_oracle(p, pool[:per_step], threads=threads)
        times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = per_step * args.steps / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000 * tot / args.steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3: batch of 1024x440 frames, w=5, D=128 (bounded sample: "
                               f"{per_step} frames per step)", "frames_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "oracle",
                         "sample": f"{per_step} frames per step, oracle prefix mode, "
                                   f"{threads} threads"},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


SWEEP = [  # (W, H, s, D): C4 stixel widths, then resolutions at s=5 (fig:fps)
    (1024, 440, 3, 128), (1024, 440, 5, 128), (1024, 440, 7, 128), (1024, 440, 10, 128),
    (512, 440, 5, 128), (2048, 440, 5, 128),             # width: linear
    (1024, 220, 5, 128), (1024, 880, 5, 128),             # height: quadratic
    (640, 480, 5, 128), (1280, 480, 5, 128),              # the paper's quoted 1280x480
    (2048, 1024, 5, 256),                                  # C5 (per GPU)
]


def run_sweep(args, local):
    """NEXT f1: fps and fps/W over resolutions and stixel widths,
    each config with sampled exact parity against the oracle.  Power is the
    median nvidia-smi power.draw during the timed region."""
    import torch
    from paper_1610_04124_b200 import stixels as S
    from inputs import synth
    from oracle import oracle as orc
    from tests import modelparams as mp
    from tests.gpuharness import compare_exact
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    lines = []
    for (W, H, s, D) in SWEEP:
        p = mp.make(max_disparity=D, stixel_width=s,
                    ground_slope=0.35 if D == 256 else 0.4)
        if D == 256:
            p["cost_frac_bits"] = 10                          # L#22: q=10 for C5
        cells = (W // s) * H * (H + 1) // 2
        B = int(max(16, min(4096, 0.2 * 4e11 / cells)))     # ~0.2 s per batch at ~4e11 cells/s
        nd = min(16, B)
        pool = np.stack([synth.frame(4, i, W, H, D, alpha=p["ground_slope"]) for i in range(nd)])
        disp = torch.from_numpy(pool.view(np.int16)).to(dev)[torch.arange(B) % nd]
        hd = S.Handle(S.params_from_dict(p, H), W, H, B, device=local, stream=stream)
        out, cnt, cost = hd.alloc_outputs(B)
        with torch.cuda.stream(stream):
            for _ in range(max(3, args.warmup)):
                hd.compute(disp, out, cnt, cost)
        torch.cuda.synchronize()
        # sampled parity: 2 frames x 6 columns
        m = mp.oracle_model(p, H)
        rng = np.random.default_rng(W + H + s)
        got = S.decode(out[:2].cpu().numpy(), cnt[:2].cpu().numpy())
        ch = cost[:2].cpu().numpy()
        bad = 0
        for f in range(2):
            ci = rng.choice(hd.n_cols, 6, replace=False)
            rc = orc.reduce(pool[f], s, 4, 0xFFFF, D)[ci]
            st, oc = orc.solve_frame(m, rc)
            bad += len(compare_exact([[got[f][c] for c in ci]], [ch[f][ci]], [st], [oc],
                                     p["cost_frac_bits"]))
        steps = max(3, args.steps)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sampler = ClockSampler(local)
        sampler.start()
        time.sleep(0.3)
        with torch.cuda.stream(stream):
            e0.record(stream)
            for _ in range(steps):
                hd.compute(disp, out, cnt, cost)
            e1.record(stream)
        torch.cuda.synchronize()
        clocks = sampler.stop()
        ms = e0.elapsed_time(e1) / steps
        fps = B / (ms / 1000.0)
        line = {"sweep": "f1", "W": W, "H": H, "s": s, "D": D, "batch": B, "fps": fps,
                "ms_per_batch": ms, "cells_per_s": cells * fps,
                "power_w": clocks.get("power_w"),
                "fps_per_watt": fps / clocks["power_w"] if clocks.get("power_w") else None,
                "clocks": clocks,
                "parity": "exact (12 sampled columns)" if bad == 0 else f"MISMATCH {bad}/12"}
        lines.append(line)
        print(json.dumps(line), flush=True)
        hd.destroy()
        del disp
    if args.sweep_out:
        with open(args.sweep_out, "w") as fo:
            for line in lines:
                fo.write(json.dumps(line) + "\n")


def run_quality(n, local):
    """NEXT f3: detection rate and false positives of the
    CUDA path's stixels on n noisy C2-distribution frames (config 5 seeds)
    against the scenes' ground truth (paper_1610_04124_b200/quality.py), for the
    mean and the median (f4) column reduction."""
    import torch
    from paper_1610_04124_b200 import quality as Q
    from paper_1610_04124_b200 import stixels as S
    from inputs import synth
    dev = torch.device("cuda", local)
    scenes = [synth.random_scene(5000 + i, W_IMG, H_IMG, D_MAX) for i in range(n)]
    frames = np.stack([synth.render(sc, 5000 + i) for i, sc in enumerate(scenes)])
    labs = [Q.column_labels(synth.gt_labels(sc), S_W) for sc in scenes]
    disp = torch.from_numpy(frames.view(np.int16)).to(dev)
    res = {}
    for name, mode in (("mean", S.REDUCE_MEAN), ("median", S.REDUCE_MEDIAN)):
        p = dict(params_dict(), reduce_mode=mode)
        hd = S.Handle(S.params_from_dict(p, H_IMG), W_IMG, H_IMG, n, device=local)
        out, cnt, cost = hd.alloc_outputs(n)
        hd.compute(disp, out, cnt, cost)
        hd.sync()
        lists = S.decode(out.cpu().numpy(), cnt.cpu().numpy())
        res[name] = Q.summarize([Q.evaluate_frame(lists[b], labs[b], S_W) for b in range(n)])
        hd.destroy()
    line = {"quality": "f3", "workload": f"{n} noisy C2 frames (1024x440, w=5, D=128), "
                                         "ground truth from the synthetic scenes",
            "reduce_mean": res["mean"], "reduce_median": res["median"],
            "paper_context": "Table 1 (P:261-273): 88.7% detection, 2.14% pairs with FP, 155 FP "
                             "on 1495 real pairs (not comparable: synthetic scenes here)"}
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    rank, world, local = dist_env()
    import torch
    import torch.distributed as dist
    if world > 1 and not dist.is_initialized():
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    assert torch.cuda.is_available(), "bench.py (ours) needs a GPU"
    torch.cuda.set_device(local)
    from paper_1610_04124_b200 import build as b
    b.build()
    from paper_1610_04124_b200 import stixels as S
    if args.sweep:
        if rank == 0:
            run_sweep(args, local)
        return
    if args.quality:
        if rank == 0:
            run_quality(args.quality, local)
        return

    p = params_dict()
    B = args.batch
    pool = frame_pool(min(args.distinct, B), rank)
    idx = np.arange(B) % len(pool)
    dev = torch.device("cuda", local)
    stream = torch.cuda.Stream(dev)
    disp = torch.empty((B, H_IMG, W_IMG), dtype=torch.int16, device=dev)
    pool_t = torch.from_numpy(pool.view(np.int16)).to(dev)
    disp.copy_(pool_t[torch.from_numpy(idx).to(dev)])
    del pool_t
    params = S.params_from_dict(p, H_IMG)
    hd = S.Handle(params, W_IMG, H_IMG, B, device=local, stream=stream)
    dp_variant = hd.dp_variant
    out, cnt, cost = hd.alloc_outputs(B)
    cols = torch.empty((B, hd.n_cols, H_IMG), dtype=torch.int16, device=dev)
    torch.cuda.synchronize()

    def step(evs=None):
        with torch.cuda.stream(stream):
            if evs:
                evs[0].record(stream)
            hd.reduce(disp, cols)
            if evs:
                evs[1].record(stream)
            hd.solve(cols, out, cnt, cost)
            if evs:
                evs[2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()

    # sampled parity against the oracle at full size, same launch configuration
    parity = "skipped"
    if rank == 0:
        from tests.gpuharness import compare_exact
        from oracle import oracle as orc
        from tests import modelparams as mp
        rng = np.random.default_rng(1)
        fr = rng.choice(B, 4, replace=False)
        m = mp.oracle_model(p, H_IMG)
        out_h, cnt_h, cost_h = out[fr].cpu().numpy(), cnt[fr].cpu().numpy(), cost[fr].cpu().numpy()
        got = S.decode(out_h, cnt_h)
        bad = 0
        for i, f in enumerate(fr):
            cidx = rng.choice(hd.n_cols, 8, replace=False)
            rcols = orc.reduce(pool[idx[f]], S_W, 4, 0xFFFF, D_MAX)[cidx]
            st, oc = orc.solve_frame(m, rcols)
            bad += len(compare_exact([[got[i][c] for c in cidx]], [cost_h[i][cidx]], [st], [oc],
                                     p["cost_frac_bits"]))
        parity = "exact (32 sampled columns)" if bad == 0 else f"MISMATCH on {bad}/32 columns"

    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    sampler = ClockSampler(local)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    sampler.start()
    time.sleep(0.3)
    for k in range(args.steps):
        step(evs[k])
    torch.cuda.synchronize()
    clocks = sampler.stop()
    if world > 1:
        dist.barrier()
    red = [e[0].elapsed_time(e[1]) for e in evs]
    dp = [e[1].elapsed_time(e[2]) for e in evs]
    step_ms = [r + d for r, d in zip(red, dp)]
    total_ms = sum(step_ms)
    max_ms = max_over_ranks(total_ms, world, dev)
    frames_total = B * world * args.steps
    value = aggregate_value(B, args.steps, world, max_ms)

    # roofline of the dominant kernel (the DP): algorithmic ALU ops / duration
    peaks = measured_peaks()
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_tops = n_sm * 4 * 32 * sm_max * 1e6 / 1e12       # lane-instruction issue peak
    dp_ms = statistics.mean(dp)
    cells = cells_per_frame() * B
    achieved = cells * ALG_OPS_PER_CELL / (dp_ms / 1000.0) / 1e12
    prof = ncu_profile()
    tpf = prof.get("dram_bytes_per_frame")
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_tops, "unit": "Tops/s",
                "frac": achieved / peak_tops,
                "traffic": (tpf * B) if tpf is not None else None,
                "kernel": "dp_kernel", "ops_per_cell": ALG_OPS_PER_CELL,
                "cells_per_launch": cells,
                "peak_note": f"{n_sm} SMs x 128 lanes x {sm_max:.0f} MHz (issue peak, "
                             "B200_PROFILING/B300_MICROARCH unit counts; DESIGN.md 5b)",
                "ncu_pipe_util": prof.get("pipe_util")}
    # K1 (a1-a2) against HBM: algorithmic bytes = input read + reduced columns written
    red_ms = statistics.mean(red)
    red_bytes = B * (W_IMG * H_IMG * 2 + (W_IMG // S_W) * H_IMG * 2)
    hbm_peak = peaks.get("hbm_gbs", 6555.2)
    k1_roofline = {"bound": "hbm", "kernel": "reduce_kernel", "unit": "GB/s",
                   "achieved": red_bytes / (red_ms / 1000.0) / 1e9, "peak": hbm_peak,
                   "frac": red_bytes / (red_ms / 1000.0) / 1e9 / hbm_peak,
                   "bytes_per_launch": red_bytes}

    # end-to-end through the C ABI with host buffers (pinned), copies included
    e2e = None
    if not args.no_e2e:
        eb = min(args.e2e_batch, B)
        p2 = dict(p, max_stixels=128)
        hd2 = S.Handle(S.params_from_dict(p2, H_IMG), W_IMG, H_IMG, min(eb, 32), device=local,
                       stream=stream)
        hin = torch.empty((eb, H_IMG, W_IMG), dtype=torch.int16).pin_memory()
        hin.copy_(torch.from_numpy(pool[idx[:eb]].view(np.int16)))
        hout = torch.empty((eb, hd2.n_cols, hd2.cap, 12), dtype=torch.uint8).pin_memory()
        hcnt = torch.empty((eb, hd2.n_cols), dtype=torch.int32).pin_memory()
        hcost = torch.empty((eb, hd2.n_cols), dtype=torch.float32).pin_memory()
        pitch = W_IMG * 2
        hd2.compute_host_ptr(hin.data_ptr(), pitch, eb, hout.data_ptr(), hcnt.data_ptr(),
                             hcost.data_ptr())
        e_steps = max(1, min(args.steps, 3))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            hd2.compute_host_ptr(hin.data_ptr(), pitch, eb, hout.data_ptr(), hcnt.data_ptr(),
                                 hcost.data_ptr())
        dt = max_over_ranks(time.perf_counter() - t0, world, dev)
        e2e = {"value": world * eb * e_steps / dt, "unit": "frames/s",
               "h2d_bytes_per_step": eb * H_IMG * pitch,
               "d2h_bytes_per_step": eb * hd2.n_cols * (hd2.cap * 12 + 8),
               "frames_per_step": eb, "max_stixels": 128,
               "note": "stixels_compute_host: pinned host buffers, ~32-frame stages (29 at 1024x440) on 2 "
                       "streams, synchronous call; wall clock max over ranks"}
        hd2.destroy()

    # BASELINE configs[1]: ONE frame per call (latency; the GPU is mostly idle: 204
    # columns for 592 column slots), frames back to back, inputs resident
    single = None
    if rank == 0 and not args.no_single:
        hd1 = S.Handle(params, W_IMG, H_IMG, 1, device=local, stream=stream)
        o1, c1, k1 = hd1.alloc_outputs(1)
        with torch.cuda.stream(stream):
            for i in range(3):
                hd1.compute(disp[i:i + 1], o1, c1, k1)
        torch.cuda.synchronize()
        n1 = 50
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            s0.record(stream)
            for i in range(n1):
                hd1.compute(disp[i:i + 1], o1, c1, k1)
            s1.record(stream)
        torch.cuda.synchronize()
        lat_ms = s0.elapsed_time(s1) / n1
        single = {"workload": "configs[1]: single 1024x440 frame per call (w=5, D=128)",
                  "latency_us": 1000.0 * lat_ms, "fps": 1000.0 / lat_ms, "calls": n1}
        hd1.destroy()

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(p, pool, args.cpu_frames)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": max_ms / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "i32" if dp_variant == S.DP_INT32 else "f32",
            "dtype_note": ("exact-mode cost quanta (2^-q nat, L#22): int32 in the rectangle cells, "
                           "integer-valued fp32 in the serial triangle chain"
                           if dp_variant == S.DP_INT32 else "exact-mode cost quanta in fp32 (L#22)"),
            "data": "synthetic",
            "config": {"workload": f"C3: batch of {B} frames 1024x440 per GPU, w=5, D=128, "
                                   "u16 disparities (4 frac bits), exact-mode costs q=11",
                       "frames_per_gpu_per_step": B, "distinct_seeded_frames": len(pool),
                       "l2": "inputs 3.7 GB per step >> 126 MB L2 (no flush needed)",
                       "parallelism": f"frames sharded over {world} GPU(s), no collective",
                       "dp_kernel": {S.DP_DENSE: "fp32 dense W-row ring", S.DP_SPARSE: "fp32 sparse bands",
                                     S.DP_PAIR2D: "fp32 f2 tables",
                                     S.DP_INT32: "int32 quanta, atomic band rounds"}[dp_variant]},
            "cells_per_s": cells_per_frame() * frames_total / (max_ms / 1000.0),
            "stage_ms": {"reduce": statistics.mean(red), "dp": dp_ms},
            "stage_share": {"reduce": sum(red) / total_ms, "dp": sum(dp) / total_ms},
            "roofline": roofline, "k1_roofline": k1_roofline, "cpu_baseline": cpu, "e2e": e2e,
            "single_frame": single,
            "gpu_launches": 2 * args.steps, "clocks": clocks, "parity": parity,
            "fps_per_watt": (value / world / clocks["power_w"]) if clocks.get("power_w") else None,
        }
        print(json.dumps(line), flush=True)
    hd.destroy()
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
