"""Multi-process host logic of bench.py on CPU (gloo, world size 2): frames are
sharded with disjoint seeds per rank (weak scaling, no data-path collective) and
timing is the max over ranks."""
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
    r, w, local = bench.dist_env()
    assert (r, w, local) == (rank, world, rank)
    seeds = bench.frame_indices(rank, 8)
    gathered = [None] * world
    dist.all_gather_object(gathered, seeds)
    # per-rank "device time": rank 1 is slower; the job time is the max
    ms = 100.0 + 50.0 * rank
    m = bench.max_over_ranks(ms, world)
    v = bench.aggregate_value(4096, 5, world, m)
    out[rank] = (gathered, m, v)
    dist.barrier()
    dist.destroy_process_group()


def test_sharding_and_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    manager = mp.Manager()
    out = manager.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    g0, m0, v0 = out[0]
    g1, m1, v1 = out[1]
    assert set(g0[0]).isdisjoint(g0[1])          # disjoint frames per rank
    assert g0 == g1
    assert m0 == m1 == 150.0                     # slowest rank
    assert v0 == v1 == pytest.approx(4096 * 2 * 5 / 0.150)
