"""Multi-process (gloo, world_size 2) checks of the multi-GPU decomposition on CPU.

The GPU path shards one signal into contiguous output ranges with a (k-1)-sample halo
(or a batch into rows); every rank filters its slice independently and the only
collective is the final gather.  Here each rank runs the CPU oracle on
its slice, the pieces are gathered over gloo, and the result must equal the unsharded
output bit for bit.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, k, n, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1406_1717_b200.shard as sh
        from oracle_lib import Oracle
        orc = Oracle()
        rng = np.random.default_rng(123)
        x = rng.standard_normal(n).astype(np.float32)          # every rank builds the same signal
        shard = sh.shard_outputs(n, k, world)[rank]
        part = sh.run_shard(x, k, shard, orc.median_filter)    # rank-local filter, no exchange
        full = sh.gather_outputs([part], world, rank, dist=dist)
        # fold_checksum of the global output, chained over ranks in rank order
        cks = sh.chained_fold_checksum(part, world, rank, dist=dist)
        # rows: shard whole rows, gather
        xr = rng.integers(0, 16, size=(7, 3 * k + 5)).astype(np.int32)
        r0, r1 = sh.shard_rows(xr.shape[0], world)[rank]
        rows_part = np.stack([orc.median_filter(xr[r], k) for r in range(r0, r1)]) if r1 > r0 else \
            np.zeros((0, xr.shape[1] - k + 1), np.int32)
        rows_full = sh.gather_outputs([rows_part], world, rank, dist=dist)
        if rank == 0:
            want = orc.median_filter(x, k)
            want_rows = np.stack([orc.median_filter(xr[r], k) for r in range(xr.shape[0])])
            q.put((bool(np.array_equal(full.view(np.int32), want.view(np.int32))),
                   bool(np.array_equal(rows_full, want_rows)),
                   cks == orc.fold_checksum(want)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,n,world", [(3, 1000, 2), (31, 5003, 2), (255, 20000, 2), (2049, 30011, 2),
                                       (101, 7001, 3)])
def test_sharded_equals_unsharded_gloo(k, n, world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, k, n, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    ok_signal, ok_rows, ok_cks = q.get(timeout=10)
    assert ok_signal and ok_rows and ok_cks


def test_shard_plan_properties():
    import paper_1406_1717_b200.shard as sh
    for n, k, world in [(100, 3, 8), (10, 9, 4), (5, 7, 2), (10**6, 101, 8), (2**20 + 3, 1023, 3)]:
        shards = sh.shard_outputs(n, k, world)
        keep = max(n - k + 1, 0)
        assert shards[0].out_begin == 0 and shards[-1].out_end == keep
        for a, b in zip(shards, shards[1:]):
            assert a.out_end == b.out_begin
        for s in shards:
            if s.n_out:
                assert s.n_in == s.n_out + k - 1 and s.in_end <= n
    assert sh.shard_rows(10, 4) == [(0, 2), (2, 5), (5, 7), (7, 10)]


def test_fold_checksum_matches_reference_and_chains():
    """mf_fold_checksum (product library, host) == the oracle's fold_checksum (io.hpp:17-28)
    for every dtype, and folding a continuation from a previous state equals folding the
    concatenation (what the multi-rank bench relies on)."""
    import paper_1406_1717_b200 as mf
    from oracle_lib import Oracle
    orc = Oracle()
    rng = np.random.default_rng(5)
    for dt in (np.int32, np.int64, np.float32, np.float64):
        v = (rng.standard_normal(1001) * 1e3).astype(dt)
        assert mf.fold_checksum(v) == orc.fold_checksum(v)
        for cut in (0, 1, 500, 1001):
            assert mf.fold_checksum(v[cut:], mf.fold_checksum(v[:cut])) == mf.fold_checksum(v)
