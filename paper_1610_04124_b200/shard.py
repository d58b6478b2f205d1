"""Frame sharding across GPUs (BASELINE configs[2]).

Columns -- and therefore frames -- are independent ("stixels in different
columns are independent"), so a batch of frames splits into contiguous
per-rank shards with no exchange on the data path: one process per GPU, each
with its own handle, stream, tables and inputs.  The only collectives are
host-side bookkeeping after the timed region: the max-over-ranks timing and an
optional gather of the (small) outputs to rank 0, over whatever backend the
process group uses (NCCL between B200s, gloo on CPU).  This module is
argument/index plumbing only; every step of the hot path runs in libstixels.so.
"""
from __future__ import annotations


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) of `n` frames owned by `rank` of `world`; the
    first n % world ranks take one frame more.  Shards tile [0, n) in rank order."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank / world size")
    base, rem = divmod(n, world)
    start = rank * base + min(rank, rem)
    return start, start + base + (1 if rank < rem else 0)


def gather_shards(t, n: int, rank: int, world: int):
    """All-gather a rank's shard `t` ([shard frames, ...], on the backend's device)
    into the full [n, ...] batch in frame order (returned on every rank).  Shards
    may differ in length by one frame: each is padded to the longest first."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return t
    sizes = [shard_range(n, r, world) for r in range(world)]
    mx = max(b - a for a, b in sizes)
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad)
    return torch.cat([parts[r][: b - a] for r, (a, b) in enumerate(sizes)], dim=0)
