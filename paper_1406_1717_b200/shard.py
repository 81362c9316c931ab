"""Multi-GPU decomposition: contiguous output ranges with a (k-1)-sample halo, or rows.

A single signal's n-k+1 outputs are cut into G contiguous ranges [o_g, o_{g+1});
rank g filters the input slice x[o_g, o_{g+1} + k - 1) as an independent signal.
Blocking never changes an output (every median is the (h+1)-th smallest of its own
window), so the concatenation is bit-identical to the unsharded
run.  Batches shard whole rows.  There is no exchange step during compute; the only
collective is the optional final gather, a device gather onto one rank (NCCL send/recv
over NVLink under torch.distributed's ``gather``), or -- in one process -- the per-device
D2H into the host output at offset o_g (``Context.multi``, mf_context_create_multi).
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


def input_union(n: int, ks, world: int, rank: int) -> tuple[int, int]:
    """[begin, end) of the global input rank `rank` needs to serve its shard for every
    window in `ks`: the union of the per-k ranges [o_g, o_{g+1} + k - 1).  The output
    split depends on k, so a single buffer must cover the smallest begin and the largest
    end over all k (sizing it from one k leaves the others short)."""
    spans = [shard_outputs(n, k, world)[rank] for k in ks]
    spans = [s for s in spans if s.n_out > 0] or spans[:1]
    return min(s.in_begin for s in spans), max(s.in_end for s in spans)


def shard_view(x, begin: int, shard: Shard):
    """Rank-local input slice of `shard` inside a buffer holding global samples
    [begin, begin + len(x)); raises if the buffer does not cover the shard."""
    a = shard.in_begin - begin
    if a < 0 or a + shard.n_in > len(x):
        raise ValueError(f"input buffer [{begin}, {begin + len(x)}) does not cover shard "
                         f"[{shard.in_begin}, {shard.in_end})")
    return x[a:a + shard.n_in]


def shard_rows(rows: int, world: int) -> list[tuple[int, int]]:
    """Contiguous row ranges [r0, r1) per rank."""
    return [(rows * g // world, rows * (g + 1) // world) for g in range(world)]


def run_shard(x, k: int, shard: Shard, filt):
    """Filter rank `shard.rank`'s slice with `filt(slice, k)` (the CUDA entry in production)."""
    if shard.n_out == 0:
        return x[:0]
    return filt(x[shard.in_begin:shard.in_end], k)


def gather_outputs_device(part, world: int, rank: int, dist=None, dst: int = 0):
    """Final gather of per-rank output ranges (torch tensors, 1-D or rows x len) onto
    rank `dst`: one ``dist.gather`` of equal-size tensors -- under NCCL a grouped
    send/recv straight between device buffers over NVLink, under gloo host tensors -- then
    a trim and a concatenation on `dst`'s device.  Returns the concatenation on `dst`,
    None elsewhere.  Single process: returns `part`."""
    import torch
    if dist is None or world == 1:
        return part
    # per-rank lengths (leading dimension) first, so every rank sends one padded tensor
    lens = torch.tensor([part.shape[0]], dtype=torch.int64, device=part.device)
    all_lens = [torch.zeros_like(lens) for _ in range(world)]
    dist.all_gather(all_lens, lens)
    all_lens = [int(t.item()) for t in all_lens]
    cap = max(all_lens)
    buf = torch.empty((cap,) + tuple(part.shape[1:]), dtype=part.dtype, device=part.device)
    buf[:part.shape[0]].copy_(part)
    bufs = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, bufs, dst=dst)
    if rank != dst:
        return None
    return torch.cat([b[:n] for b, n in zip(bufs, all_lens)])


def gather_outputs(parts, world: int, rank: int, dist=None, dst: int = 0):
    """numpy front end of ``gather_outputs_device`` (host arrays, gloo): the concatenation
    on `dst`, None elsewhere."""
    import numpy as np
    import torch
    if dist is None or world == 1:
        return np.concatenate([np.asarray(p) for p in parts])
    out = gather_outputs_device(torch.from_numpy(np.ascontiguousarray(parts[0])), world, rank, dist=dist, dst=dst)
    return None if out is None else out.numpy()


def chained_fold_checksum(part, world: int, rank: int, dist=None, fold=None):
    """fold_checksum (io.hpp:17-28) of the concatenation of every rank's outputs: FNV-1a
    is sequential but chainable, so rank r folds its part starting from rank r-1's state
    (point-to-point over `dist`) and the last rank sends the result to rank 0.  Returns
    the global checksum on rank 0 (None elsewhere).  `part` is a host array."""
    import torch
    from .filter import fold_checksum
    from ._native import MF_FOLD_INIT
    fold = fold or fold_checksum
    if dist is None or world == 1:
        return fold(part, MF_FOLD_INIT)
    dev = "cpu" if dist.get_backend() == "gloo" else f"cuda:{torch.cuda.current_device()}"
    state = torch.tensor([MF_FOLD_INIT], dtype=torch.int64, device=dev)  # uint64 bits as int64
    if rank > 0:
        dist.recv(state, src=rank - 1)
    h = fold(part, int(state.item()) & ((1 << 64) - 1))
    out = torch.tensor([h - (1 << 64) if h >= 1 << 63 else h], dtype=torch.int64, device=dev)
    if rank < world - 1:
        dist.send(out, dst=rank + 1)
    elif rank != 0:
        dist.send(out, dst=0)
    if rank == 0:
        if world > 1:
            dist.recv(out, src=world - 1)
        return int(out.item()) & ((1 << 64) - 1)
    return None
