"""Multi-GPU decomposition: contiguous output ranges with a (k-1)-sample halo, or rows.

A single signal's n-k+1 outputs are cut into G contiguous ranges [o_g, o_{g+1});
rank g filters the input slice x[o_g, o_{g+1} + k - 1) as an independent signal.
Blocking never changes an output (every median is the (h+1)-th smallest of its own
window), so the concatenation is bit-identical to the unsharded
run.  Batches shard whole rows.  There is no exchange step during compute; the only
collective is the optional final gather.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Shard:
    rank: int
    out_begin: int   # o_g
    out_end: int     # o_{g+1}
    in_begin: int    # o_g
    in_end: int      # o_{g+1} + k - 1

    @property
    def n_out(self) -> int:
        return self.out_end - self.out_begin

    @property
    def n_in(self) -> int:
        return self.in_end - self.in_begin


def shard_outputs(n: int, k: int, world: int) -> list[Shard]:
    """Balanced contiguous output ranges (the same split as the CPU baseline harness)."""
    if world < 1:
        raise ValueError("world must be >= 1")
    keep = n - k + 1 if n >= k else 0
    shards = []
    for g in range(world):
        o0 = keep * g // world
        o1 = keep * (g + 1) // world
        shards.append(Shard(g, o0, o1, o0, (o1 + k - 1) if o1 > o0 else o0))
    return shards


def shard_rows(rows: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges [r0, r1) per rank."""
    return [(rows * g // world, rows * (g + 1) // world) for g in range(world)]


def run_shard(x, k: int, shard: Shard, filt):
    """Filter rank `shard.rank`'s slice with `filt(slice, k)` (the CUDA entry in production)."""
    if shard.n_out == 0:
        return x[:0]
    return filt(x[shard.in_begin:shard.in_end], k)


def gather_outputs(parts, world: int, rank: int, dist=None, dst: int = 0):
    """Final gather of per-rank output ranges onto `dst` (torch.distributed object gather).

    Returns the concatenation on `dst`, None elsewhere.  Single process: concatenates."""
    import numpy as np
    if dist is None or world == 1:
        return np.concatenate([np.asarray(p) for p in parts])
    objs = [None] * world if rank == dst else None
    dist.gather_object(np.asarray(parts[0]), objs, dst=dst)
    if rank != dst:
        return None
    return np.concatenate(objs)
