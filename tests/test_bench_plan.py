"""CPU checks of bench.py's multi-GPU input plan: for every config and world size each
rank's single input buffer covers its halo'd shard for EVERY k of the config (the round-1
bench sized it from the smallest k, so ranks >= 1 silently filtered truncated views)."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_1406_1717_b200.shard import shard_outputs, shard_view  # noqa: E402


@pytest.mark.parametrize("world", [1, 2, 4, 8])
@pytest.mark.parametrize("cfg", ["c1", "c2", "c4", "c5"])
def test_every_rank_view_holds_its_shard(cfg, world):
    dtype, n, ks, gen, seed, rows = bench.CONFIGS[cfg]
    total_out = {k: 0 for k in ks}
    for rank in range(world):
        begin, end = bench.input_range(cfg, rank, world)
        assert 0 <= begin < end <= n * world
        x = range(begin, end)                           # global sample index per slot (lazy)
        for k in ks:
            sh = shard_outputs(n * world, k, world)[rank]
            v, n_out = bench.shard_views(cfg, x, begin, rank, world, k)
            assert len(v) == sh.n_in == n_out + k - 1
            assert v[0] == sh.in_begin and v[-1] == sh.in_end - 1
            total_out[k] += n_out
        # the buffer is no wider than the union of the shards
        assert begin == min(shard_outputs(n * world, k, world)[rank].in_begin for k in ks)
        assert end == max(shard_outputs(n * world, k, world)[rank].in_end for k in ks)
    for k in ks:
        assert total_out[k] == n * world - k + 1


def test_shard_view_rejects_short_buffer():
    sh = shard_outputs(1000, 31, 2)[1]
    x = np.arange(sh.in_begin + 5, 1000)
    with pytest.raises(ValueError):
        shard_view(x, sh.in_begin + 5, sh)


def test_rows_plan_covers_all_rows():
    import paper_1406_1717_b200 as mf
    for world in (1, 2, 4, 8):
        got = [r for a, b in mf.shard_rows(4096 * world, world) for r in range(a, b)]
        assert got == list(range(4096 * world))
