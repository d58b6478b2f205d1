#!/usr/bin/env python
"""Benchmark of the stixel hot path (BASELINE.json metric: frames/s at
1024x440 w=5 on 1/2/4/8 B200; DP cell-updates/s vs pipe peak).

One step = one pass of the whole hot path (reduction + DP + backtracking,
SURVEY 8(a) a1-a7) over one batch of synthetic frames resident in HBM:
config C3 (BASELINE configs[2]), 4096 frames of 1024x440, w=5, D=128, split
into contiguous 4096/N shards over N GPUs (strong scaling; `--weak` gives every
rank its own 4096).  Frames are independent, so there is no collective
on the data path; the process group carries only barriers, the max-over-ranks
timing and, after the timed region, a gather of per-frame output digests (the
cross-rank identity check of SURVEY 8(e)).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Rank 0 prints ONE JSON line.  `--impl reference` times the CPU oracle (the
reference arm for this paper-only tier) on the host cores; `--cpu-full` runs
BASELINE.md's oracle plan (C1-C5 samples) and prints its own line.
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
    ap.add_argument("--batch", type=int, default=4096,
                    help="frames per step for the whole job (BASELINE configs[2]: 4096, split "
                         "4096/N over N GPUs); with --weak: frames per rank")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: every rank runs its own --batch frames")
    ap.add_argument("--distinct", type=int, default=128, help="distinct seeded frames in the pool")
    ap.add_argument("--e2e-batch", type=int, default=4096,
                    help="frames per e2e call (whole job; default: the configs[2] step, 4096)")
    ap.add_argument("--e2e-seconds", type=float, default=1.0, help="minimum e2e timed span")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cont", action="store_true", help="skip the continuous-mode (q=0) leg")
    ap.add_argument("--no-single", action="store_true", help="skip the one-frame latency run")
    ap.add_argument("--cpu-frames", type=int, default=0, help="oracle sample size (0 = auto)")
    ap.add_argument("--cpu-full", action="store_true",
                    help="only the oracle baseline plan of BASELINE.md (C1-C5 samples, 1 thread "
                         "and all cores; one JSON line, no GPU)")
    ap.add_argument("--lib", default="", help="time another build of the same C ABI (A/B)")
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


def frame_pool(n):
    """The pool of distinct seeded C3 frames (config 3, seeds 3000 + i); global
    frame g of a step is pool frame g mod n."""
    from inputs import synth
    return np.stack([synth.frame(3, i, W_IMG, H_IMG, D_MAX) for i in range(n)])


def frame_shard(total, rank, world, weak):
    """Global frame indices [g0, g1) of this rank: a contiguous 1/N shard of the
    job's batch (strong scaling, configs[2]), or a whole batch per rank (weak)."""
    from paper_1610_04124_b200.shard import shard_range
    if weak:
        return rank * total, (rank + 1) * total
    return shard_range(total, rank, world)


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


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def _oracle_fps(p, frames, threads, W=W_IMG, H=H_IMG):
    """Frames/s of the oracle (prefix mode, reduction included) on `frames`, and
    the per-frame seconds."""
    from tests.gpuharness import run_oracle
    per = []
    for f in frames:
        t0 = time.perf_counter()
        run_oracle(p, f[None], threads=threads)
        per.append(time.perf_counter() - t0)
    return len(per) / sum(per), per


def cpu_baseline(p, pool, frames_req=0):
    """The oracle (prefix mode, OpenMP over columns, all host cores) on a bounded
    sample of the same workload; plus BASELINE.md's C2 figures: the median of 3
    frames on all cores and on ONE thread (SPEC S:583 bound: < 1 s per frame)."""
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
    _, all3 = _oracle_fps(p, pool[:3], threads)
    _, one3 = _oracle_fps(p, pool[:3], 1)
    return {"value": n / dt, "unit": "frames/s", "cores": threads, "kind": "oracle",
            "cpu_model": cpu_model(), "os_cpu_count": os.cpu_count(),
            "sample": f"{n} frames of C3 (1024x440, w=5, D=128{'; the pool of ' + str(len(pool)) + ' repeated' if n > len(pool) else ''}), oracle prefix mode O(h^2), "
                      f"double precision, OpenMP over columns, {threads} threads, {dt:.1f} s",
            "c2_median_of_3": {"all_cores_s_per_frame": statistics.median(all3),
                               "all_cores_fps": 1.0 / statistics.median(all3),
                               "one_thread_s_per_frame": statistics.median(one3),
                               "one_thread_fps": 1.0 / statistics.median(one3),
                               "spec_bound_one_thread_lt_1s": statistics.median(one3) < 1.0},
            "paper_context": "13.3 fps on a 6-core i7-980X (P:287), other hardware"}


def run_cpu_full():
    """BASELINE.md's oracle plan: C1, C2 (median of 3), C3 (64 frames,
    extrapolated), C4 (w = 3/5/7/10, 3 frames each), C5 (2 frames), on all host
    cores, C2 also on one thread.  One JSON line (kept under profiles/)."""
    from inputs import synth
    from oracle import oracle as orc
    from tests import modelparams as mp
    threads = orc.max_threads()
    res = {"cpu_baseline_plan": "BASELINE.md", "cpu_model": cpu_model(), "threads": threads,
           "os_cpu_count": os.cpu_count(), "mode": "oracle prefix O(h^2), double, OpenMP over columns"}
    sc = synth.c1_scene()
    c1 = np.stack([synth.render(sc, 1, noise=False)] * 3)
    fps, per = _oracle_fps(mp.make(max_disparity=32, ground_slope=sc.alpha), c1, threads)
    res["C1"] = {"fps": fps, "s_per_frame_median": statistics.median(per)}
    p = mp.make()
    pool = frame_pool(8)
    for th, key in ((threads, "C2_all_cores"), (1, "C2_one_thread")):
        fps, per = _oracle_fps(p, pool[:3], th)
        res[key] = {"s_per_frame_median": statistics.median(per), "fps_median": 1 / statistics.median(per),
                    "frames": 3, "threads": th}
    from tests.gpuharness import run_oracle
    t0 = time.perf_counter()
    run_oracle(p, pool[np.arange(64) % 8], threads=threads)
    dt = time.perf_counter() - t0
    res["C3"] = {"fps": 64 / dt, "frames_timed": 64,
                 "batch_4096_s_extrapolated": 4096 * dt / 64, "note": "extrapolated from 64 frames"}
    for s in (3, 5, 7, 10):
        pc = mp.make(stixel_width=s)
        fps, per = _oracle_fps(pc, pool[:3], threads)
        res[f"C4_w{s}"] = {"fps": fps, "s_per_frame_median": statistics.median(per), "frames": 3}
    p5 = mp.make(max_disparity=256, ground_slope=0.35, cost_frac_bits=10)
    c5 = np.stack([synth.frame(5, i, 2048, 1024, 256, alpha=0.35) for i in range(2)])
    fps, per = _oracle_fps(p5, c5, threads)
    res["C5"] = {"fps": fps, "s_per_frame_median": statistics.median(per), "frames": 2,
                 "W": 2048, "H": 1024, "D": 256}
    print(json.dumps(res), flush=True)


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle as it stands (the reference arm of a
    paper-only tier), on the host cores, same metric/config/unit."""
    if rank != 0:
        return
    p = params_dict()
    pool = frame_pool(4)
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
        "ms_per_step": 1000 * tot / args.steps, "higher_is_better": True,
        "scaling": "weak" if args.weak else "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "C3: batch of 1024x440 frames, w=5, D=128 (bounded sample: "
                               f"{per_step} frames per step)", "frames_per_step": per_step},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "oracle",
                         "cpu_model": cpu_model(),
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


def sampled_parity(p, S, hd, pool, pool_idx, out, cnt, cost, frames, ncols=8, seed=1):
    """Sampled columns of the given output frames against the oracle: exact mode
    -> identical lists and costs; continuous mode (q = 0) -> north_star
    tolerance (cost within 1e-4 relative, lists identical or co-optimal by
    re-score).  Returns (checked, bad)."""
    from oracle import oracle as orc
    from tests import modelparams as mp
    from tests.gpuharness import compare_exact
    rng = np.random.default_rng(seed)
    m = mp.oracle_model(p, H_IMG)
    fr = list(frames)
    out_h, cnt_h, cost_h = out[fr].cpu().numpy(), cnt[fr].cpu().numpy(), cost[fr].cpu().numpy()
    got = S.decode(out_h, cnt_h)
    bad = checked = 0
    for i, f in enumerate(fr):
        cidx = rng.choice(hd.n_cols, ncols, replace=False)
        rcols = orc.reduce(pool[pool_idx[f]], S_W, 4, 0xFFFF, D_MAX)[cidx]
        st, oc = orc.solve_frame(m, rcols)
        checked += len(cidx)
        if p["cost_frac_bits"]:
            bad += len(compare_exact([[got[i][c] for c in cidx]], [cost_h[i][cidx]], [st], [oc],
                                     p["cost_frac_bits"]))
            continue
        for j, c in enumerate(cidx):
            if abs(cost_h[i][c] - oc[j]) > 1e-4 * abs(oc[j]):
                bad += 1
            elif [(a, b, k, float(np.float32(d))) for a, b, k, d in st[j]] != got[i][c] and \
                    abs(orc.rescore(m, rcols[j], got[i][c]) - oc[j]) > 1e-4 * abs(oc[j]):
                bad += 1
    return checked, bad


def main():
    args = parse()
    rank, world, local = dist_env()
    if args.cpu_full:
        if rank == 0:
            run_cpu_full()
        return
    import torch
    import torch.distributed as dist
    if args.impl == "reference":
        if world > 1 and not dist.is_initialized():
            dist.init_process_group("gloo")
        run_reference(args, rank, world)
        if dist.is_initialized():
            dist.destroy_process_group()
        return

    assert torch.cuda.is_available(), "bench.py (ours) needs a GPU"
    # one process per GPU over NCCL.  (Only when there are fewer GPUs than ranks --
    # a multi-rank smoke run on a 1-GPU box -- do ranks share devices; NCCL cannot
    # put two ranks on one GPU, so the host bookkeeping then goes over gloo.)
    shared = torch.cuda.device_count() < world
    local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1 and not dist.is_initialized():
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    cdev = torch.device("cpu") if shared else dev      # device of collective tensors
    # build once: rank 0 rebuilds a stale library while the other ranks wait
    from paper_1610_04124_b200 import build as b
    if rank == 0:
        b.build()
    if world > 1:
        dist.barrier()
    from paper_1610_04124_b200 import stixels as S
    from paper_1610_04124_b200.shard import gather_shards
    if args.lib:
        S.use_library(args.lib)
    if args.sweep:
        if rank == 0:
            run_sweep(args, local)
        return
    if args.quality:
        if rank == 0:
            run_quality(args.quality, local)
        return

    p = params_dict()
    g0, g1 = frame_shard(args.batch, rank, world, args.weak)
    B = g1 - g0                                   # this rank's frames per step
    job_frames = args.batch * (world if args.weak else 1)
    pool = frame_pool(min(args.distinct, job_frames))
    idx = np.arange(g0, g1) % len(pool)           # pool frame of each local frame
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

    def step(h, evs=None):
        with torch.cuda.stream(stream):
            if evs:
                evs[0].record(stream)
            h.reduce(disp, cols)
            if evs:
                evs[1].record(stream)
            h.solve(cols, out, cnt, cost)
            if evs:
                evs[2].record(stream)

    def timed(h, steps, sample_clocks):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(steps)]
        sampler = ClockSampler(local)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        if sample_clocks:
            sampler.start()
            time.sleep(0.3)
        for k in range(steps):
            step(h, evs[k])
        torch.cuda.synchronize()
        clocks = sampler.stop() if sample_clocks else None
        if world > 1:
            dist.barrier()
        red = [e[0].elapsed_time(e[1]) for e in evs]
        dp = [e[1].elapsed_time(e[2]) for e in evs]
        return red, dp, clocks

    for _ in range(args.warmup):
        step(hd)
    torch.cuda.synchronize()

    # sampled parity against the oracle at full size, same launch configuration
    parity = "skipped"
    if rank == 0:
        rng = np.random.default_rng(1)
        n_chk, bad = sampled_parity(p, S, hd, pool, idx, out, cnt, cost,
                                    rng.choice(B, min(4, B), replace=False))
        parity = f"exact ({n_chk} sampled columns)" if bad == 0 else f"MISMATCH on {bad}/{n_chk} columns"

    def skipped():                     # (an A/B build via --lib may predate the counter)
        try:
            return hd.skipped_cells()
        except (AttributeError, OSError):
            return 0
    skip0 = skipped()
    red, dp, clocks = timed(hd, args.steps, True)
    skipped_per_launch = (skipped() - skip0) / args.steps
    step_ms = [r + d for r, d in zip(red, dp)]
    total_ms = sum(step_ms)
    max_ms = max_over_ranks(total_ms, world, cdev)
    steps_max = [max_over_ranks(x, world, cdev) for x in step_ms]
    value = aggregate_value(job_frames, args.steps, 1, max_ms)

    # cross-rank identity (8(e)): frames that are the same pool frame give the same
    # bytes on every rank; per-frame digests gathered over the process group
    # (NCCL at N > 1) after the timed region
    ident = None
    with torch.no_grad():
        dig = torch.empty((B, 3), dtype=torch.int64, device=dev)
        wts = torch.randint(1, 1 << 20, (hd.cap, 3), generator=torch.Generator().manual_seed(7),
                            dtype=torch.int64).to(dev)
        ar = torch.arange(hd.cap, device=dev)
        for a0 in range(0, B, 128):
            a1 = min(B, a0 + 128)
            o = out[a0:a1].view(torch.int32).view(a1 - a0, hd.n_cols, hd.cap, 3).to(torch.int64)
            mask = (ar[None, None, :] < cnt[a0:a1, :, None]).to(torch.int64)
            dig[a0:a1, 0] = (o * wts * mask[..., None]).sum((1, 2, 3))
            dig[a0:a1, 1] = cnt[a0:a1].to(torch.int64).sum(1)
            dig[a0:a1, 2] = cost[a0:a1].double().sum(1).mul(2048.0).round().to(torch.int64)
        if not args.weak:
            full = gather_shards(dig.to(cdev), args.batch, rank, world)
            if rank == 0:
                pidx = np.arange(args.batch) % len(pool)
                fd = full.cpu().numpy()
                ok = all((fd[pidx == q] == fd[q]).all() for q in range(len(pool)))
                ident = {"check": "frames equal to the same pool frame have identical output "
                                  "digests across the whole job (all ranks gathered)",
                         "frames": args.batch, "ranks": world, "ok": bool(ok)}

    # roofline of the dominant kernel (the DP): algorithmic ALU ops / duration
    peaks = measured_peaks()
    sm_max = peaks.get("sm_max_mhz", 1965.0)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    peak_tops = n_sm * 4 * 32 * sm_max * 1e6 / 1e12       # lane-instruction issue peak
    dp_ms = statistics.mean(dp)
    cells = cells_per_frame() * B
    # `achieved` counts the algorithmic cells of the launch (every (column, target,
    # bottom) of Eq. 6).  The int32 kernel's exact chunk bound skips rectangle cells
    # whose candidates are provably worse than a known one (stixels_skipped_cells);
    # `evaluated` reports the same rate over the cells the kernel actually computed,
    # which is the measure of how the hardware is used
    evaluated = cells - skipped_per_launch
    achieved = cells * ALG_OPS_PER_CELL / (dp_ms / 1000.0) / 1e12
    ach_eval = evaluated * ALG_OPS_PER_CELL / (dp_ms / 1000.0) / 1e12
    prof = ncu_profile()
    tpf = prof.get("dram_bytes_per_frame")
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak_tops, "unit": "Tops/s",
                "frac": achieved / peak_tops,
                "traffic": (tpf * B) if tpf is not None else None,
                "kernel": "dp_kernel", "ops_per_cell": ALG_OPS_PER_CELL,
                "cells_per_launch": cells,
                "evaluated": {"cells_per_launch": evaluated, "skipped_frac": skipped_per_launch / cells,
                              "achieved": ach_eval, "frac": ach_eval / peak_tops,
                              "note": "the same rate over the cells the kernel computed (the exact "
                                      "chunk bound skips the rest)"},
                "peak_note": f"{n_sm} SMs x 128 lanes x {sm_max:.0f} MHz (issue peak, "
                             "B200_PROFILING/B300_MICROARCH unit counts; DESIGN.md 5b)",
                "ncu_pipe_util": prof.get("pipe_util")}
    # K1 (a1-a2) against HBM: algorithmic bytes = input read + reduced columns written
    red_ms = statistics.mean(red)
    red_bytes = B * (W_IMG * H_IMG * 2 + (W_IMG // S_W) * H_IMG * 2)
    hbm_peak = peaks.get("hbm_gbs", 6555.2)
    k1_roofline = {"bound": "hbm", "kernel": "reduce_strip_kernel", "unit": "GB/s",
                   "achieved": red_bytes / (red_ms / 1000.0) / 1e9, "peak": hbm_peak,
                   "frac": red_bytes / (red_ms / 1000.0) / 1e9 / hbm_peak,
                   "bytes_per_launch": red_bytes}

    # the paper-literal continuous Eq. 4 (cost_frac_bits = 0, fp32 sparse bands) on
    # the same batch: its own timing, roofline and tolerance parity
    cont = None
    if not args.no_cont:
        pc = dict(p, cost_frac_bits=0)
        hdc = S.Handle(S.params_from_dict(pc, H_IMG), W_IMG, H_IMG, B, device=local, stream=stream)
        for _ in range(args.warmup):
            step(hdc)
        torch.cuda.synchronize()
        cpar = "skipped"
        if rank == 0:
            rng = np.random.default_rng(2)
            n_chk, bad = sampled_parity(pc, S, hdc, pool, idx, out, cnt, cost,
                                        rng.choice(B, min(4, B), replace=False), seed=2)
            cpar = (f"north_star tolerance ({n_chk} sampled columns)" if bad == 0
                    else f"MISMATCH on {bad}/{n_chk} columns")
        cred, cdp, _ = timed(hdc, max(2, min(args.steps, 3)), False)
        cmax = max_over_ranks(sum(cred) + sum(cdp), world, cdev)
        cdp_ms = statistics.mean(cdp)
        cach = cells * ALG_OPS_PER_CELL / (cdp_ms / 1000.0) / 1e12
        cont = {"value": aggregate_value(job_frames, len(cdp), 1, cmax), "unit": "frames/s",
                "dtype": "f32", "cost_frac_bits": 0,
                "dp_kernel": {S.DP_SPARSE: "fp32 sparse bands", S.DP_DENSE: "fp32 dense W-row ring"}
                .get(hdc.dp_variant, str(hdc.dp_variant)),
                "ms_per_step": cmax / len(cdp),
                "roofline": {"bound": "alu", "achieved": cach, "peak": peak_tops, "unit": "Tops/s",
                             "frac": cach / peak_tops, "kernel": "dp_kernel (fp32)"},
                "parity": cpar}
        hdc.destroy()

    # end-to-end through the C ABI with host buffers (pinned), copies included,
    # timed over >= --e2e-seconds; sampled parity on its outputs
    e2e = None
    if not args.no_e2e:
        e0_, e1_ = frame_shard(args.e2e_batch, rank, world, args.weak)
        eb = e1_ - e0_
        eidx = np.arange(e0_, e1_) % len(pool)
        p2 = dict(p, max_stixels=128)
        hd2 = S.Handle(S.params_from_dict(p2, H_IMG), W_IMG, H_IMG, min(eb, 32), device=local,
                       stream=stream)
        hin = torch.empty((eb, H_IMG, W_IMG), dtype=torch.int16).pin_memory()
        hin.copy_(torch.from_numpy(pool[eidx].view(np.int16)))
        hout = torch.empty((eb, hd2.n_cols, hd2.cap, 12), dtype=torch.uint8).pin_memory()
        hcnt = torch.empty((eb, hd2.n_cols), dtype=torch.int32).pin_memory()
        hcost = torch.empty((eb, hd2.n_cols), dtype=torch.float32).pin_memory()
        pitch = W_IMG * 2

        def call():
            hd2.compute_host_ptr(hin.data_ptr(), pitch, eb, hout.data_ptr(), hcnt.data_ptr(),
                                 hcost.data_ptr())
        call()
        t0 = time.perf_counter()
        call()
        call()
        one = (time.perf_counter() - t0) / 2
        e_steps = int(max_over_ranks(max(3, int(np.ceil(1.2 * args.e2e_seconds / max(one, 1e-6)))),
                                     world, cdev))
        epar = "skipped"
        if rank == 0:
            rng = np.random.default_rng(3)
            n_chk, bad = sampled_parity(p2, S, hd2, pool, eidx, hout, hcnt, hcost,
                                        rng.choice(eb, min(3, eb), replace=False), seed=3)
            epar = f"exact ({n_chk} sampled columns)" if bad == 0 else f"MISMATCH on {bad}/{n_chk} columns"
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            call()
        dt = max_over_ranks(time.perf_counter() - t0, world, cdev)
        e2e = {"value": args.e2e_batch * (world if args.weak else 1) * e_steps / dt,
               "unit": "frames/s",
               "h2d_bytes_per_step": eb * H_IMG * pitch,
               "d2h_bytes_per_step": eb * hd2.n_cols * (hd2.cap * 12 + 8),
               "frames_per_step": eb, "steps": e_steps, "seconds": dt, "max_stixels": 128,
               "parity": epar,
               "note": "stixels_compute_host: pinned host buffers, ~32-frame stages (29 at 1024x440) on 2 "
                       "streams (own DP scratch each), synchronous call; wall clock max over ranks"}
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
                hd1.compute(disp[i % B:i % B + 1], o1, c1, k1)
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
            "ms_per_step_median": statistics.median(steps_max), "ms_per_step_min": min(steps_max),
            "ms_per_step_max": max(steps_max),
            "higher_is_better": True, "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None,
            "dtype": "i32" if dp_variant == S.DP_INT32 else "f32",
            "dtype_note": ("exact-mode cost quanta (2^-q nat, L#22): int32 in the rectangle cells, "
                           "integer-valued fp32 in the serial triangle chain"
                           if dp_variant == S.DP_INT32 else "exact-mode cost quanta in fp32 (L#22)"),
            "data": "synthetic",
            "config": {"workload": f"C3: batch of {job_frames} frames 1024x440 per step "
                                   f"({'per GPU, weak' if args.weak else f'{args.batch}/{world} per GPU'}), "
                                   "w=5, D=128, u16 disparities (4 frac bits), exact-mode costs q=11",
                       "frames_per_step": job_frames, "frames_per_gpu_per_step": B,
                       "distinct_seeded_frames": len(pool),
                       "l2": f"inputs {B * H_IMG * W_IMG * 2 / 1e9:.2f} GB per GPU per step >> 126 MB L2 "
                             "(no flush needed)",
                       "parallelism": f"contiguous frame shards over {world} GPU(s), no collective "
                                      "on the data path",
                       "dp_kernel": {S.DP_DENSE: "fp32 dense W-row ring", S.DP_SPARSE: "fp32 sparse bands",
                                     S.DP_PAIR2D: "fp32 f2 tables", S.DP_PAIR2D_DENSE: "fp32 f2 dense",
                                     S.DP_INT32: "int32 quanta, atomic band rounds"}[dp_variant],
                       "lib": args.lib or "libstixels.so",
                       "ranks_share_gpus": shared},
            "cells_per_s": cells_per_frame() * job_frames * args.steps / (max_ms / 1000.0),
            "stage_ms": {"reduce": statistics.mean(red), "dp": dp_ms},
            "stage_share": {"reduce": sum(red) / total_ms, "dp": sum(dp) / total_ms},
            "roofline": roofline, "k1_roofline": k1_roofline, "continuous": cont,
            "cpu_baseline": cpu, "e2e": e2e,
            "single_frame": single, "cross_rank_identity": ident,
            "gpu_launches": 2 * args.steps, "clocks": clocks, "parity": parity,
            "fps_per_watt": (value / world / clocks["power_w"]) if clocks.get("power_w") else None,
        }
        print(json.dumps(line), flush=True)
    hd.destroy()
    if dist.is_initialized():
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
