"""Multi-process host logic of the multi-GPU path on CPU (gloo, world size 2):
contiguous frame shards of one job batch (BASELINE configs[2]: 4096 split
4096/N), the gather of per-rank outputs back into frame order, and the
max-over-ranks timing (paper_1610_04124_b200/shard.py, bench.py)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import bench
    from paper_1610_04124_b200.shard import gather_shards, shard_range
    r, w, local = bench.dist_env()
    assert (r, w, local) == (rank, world, rank)
    n = 4097                                   # odd: shards differ by one frame
    a, b = bench.frame_shard(n, rank, world, weak=False)
    assert (a, b) == shard_range(n, rank, world)
    # a fake per-frame output that depends only on the global frame index
    shard = torch.arange(a, b, dtype=torch.int64)[:, None] * torch.tensor([[1, 7, -3]])
    full = gather_shards(shard, n, rank, world)
    # per-rank "device time": rank 1 is slower; the job time is the max
    ms = 100.0 + 50.0 * rank
    m = bench.max_over_ranks(ms, world)
    v = bench.aggregate_value(4096, 5, 1, m)
    out[rank] = ((a, b), full.numpy().tolist(), m, v, bench.frame_shard(4096, rank, world, weak=True))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_ranges_tile_the_batch():
    from paper_1610_04124_b200.shard import shard_range
    for n in (1, 7, 4096, 4097):
        for world in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(x[1] == y[0] for x, y in zip(rs, rs[1:]))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
    assert [shard_range(4096, r, 8) for r in (0, 7)] == [(0, 512), (3584, 4096)]


def test_sharding_gather_and_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    r0, f0, m0, v0, w0 = out[0]
    r1, f1, m1, v1, w1 = out[1]
    assert r0 == (0, 2049) and r1 == (2049, 4097)      # contiguous, tiling
    want = [[g, 7 * g, -3 * g] for g in range(4097)]
    assert f0 == f1 == want                            # gathered back in frame order
    assert m0 == m1 == 150.0                           # slowest rank
    assert v0 == v1 == pytest.approx(4096 * 5 / 0.150)  # job frames / job time
    assert w0 == (0, 4096) and w1 == (4096, 8192)      # --weak: a batch per rank
