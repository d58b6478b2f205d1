"""Sharded multi-process run vs one process (SURVEY.md 8(e) check): two
processes on cuda:0 (gloo process group, one handle and one stream each) run
contiguous shards of one batch; their outputs, gathered back in frame order,
are byte-identical to a single-process run of the whole batch.  (The driver
has one GPU per box; the shards here share it, which exercises the same
per-process handle / stream / shard / gather path as N GPUs.)"""
import os
import socket

import numpy as np
import pytest

from inputs import synth
from tests import modelparams as mp

pytestmark = pytest.mark.gpu

N_FRAMES, W, H = 13, 400, 220


def _frames():
    return np.stack([synth.render(synth.random_scene(6100 + i, W, H, 128), 6100 + i)
                     for i in range(N_FRAMES)])


def _run(frames, device=0):
    import torch
    from paper_1610_04124_b200 import stixels as S
    stream = torch.cuda.Stream(device)
    hd = S.Handle(S.params_from_dict(mp.make(), H), W, H, len(frames), device=device, stream=stream)
    t = torch.from_numpy(frames.view(np.int16)).cuda(device)
    out = torch.zeros((len(frames), hd.n_cols, hd.cap, 12), dtype=torch.uint8, device=f"cuda:{device}")
    cnt = torch.zeros((len(frames), hd.n_cols), dtype=torch.int32, device=f"cuda:{device}")
    cost = torch.zeros((len(frames), hd.n_cols), dtype=torch.float32, device=f"cuda:{device}")
    with torch.cuda.stream(stream):
        hd.compute(t, out, cnt, cost)
    hd.sync()
    res = out.cpu(), cnt.cpu(), cost.cpu()
    hd.destroy()
    return res


def _worker(rank, world, port, result):
    import torch
    import torch.distributed as dist
    from paper_1610_04124_b200.shard import gather_shards, shard_range
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b = shard_range(N_FRAMES, rank, world)
    out, cnt, cost = _run(_frames()[a:b])
    full = [gather_shards(x, N_FRAMES, rank, world) for x in (out, cnt, cost)]
    if rank == 0:
        result["out"] = full[0].numpy().tobytes()
        result["cnt"] = full[1].numpy().tobytes()
        result["cost"] = full[2].numpy().tobytes()
    dist.barrier()
    dist.destroy_process_group()


def test_two_process_shards_byte_identical_to_one_process():
    import torch.multiprocessing as tmp
    ref = _run(_frames())
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    manager = tmp.Manager()
    result = manager.dict()
    tmp.spawn(_worker, args=(2, port, result), nprocs=2, join=True)
    assert result["out"] == ref[0].numpy().tobytes()
    assert result["cnt"] == ref[1].numpy().tobytes()
    assert result["cost"] == ref[2].numpy().tobytes()
