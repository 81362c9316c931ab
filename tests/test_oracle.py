"""Pin the CPU oracle (oracle/medfilt_oracle.c) before trusting it (CPU only).

(a) SPEC.md known answers (tests/golden/spec_vectors.json, each re-derived from the
    reference by tests/golden/make_golden.py);
(b) the committed reference-generated fixtures (tests/golden/small_cases.npz);
(c) the reference library itself, compiled from /root/reference by oracle/Makefile,
    on seeded random inputs (skipped when oracle/_ref is absent);
(d) the reference's own exhaustive n <= 8 / {0,1,2} sweep (verify.hpp:137-178) mirrored
    against the oracle, and the naive oracle (baselines.hpp:287-300);
(e) generator recipes against the golden input checksums, and shard identity.
"""
from __future__ import annotations

import itertools
import json
import os

import numpy as np
import pytest

from oracle_lib import keymap, unkey

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "f":
        a = a.view(np.int32 if a.itemsize == 4 else np.int64)
    if b.dtype.kind == "f":
        b = b.view(np.int32 if b.itemsize == 4 else np.int64)
    return a.shape == b.shape and np.array_equal(a, b)


def test_spec_vectors(oracle):
    vec = json.load(open(os.path.join(GOLDEN, "spec_vectors.json")))
    for v in vec["median_filter"]:
        assert oracle.median_filter(np.array(v["x"], dtype=np.int64), v["k"]).tolist() == v["y"]
    for v in vec["piecewise_sort"]:
        assert oracle.piecewise_sort(np.array(v["x"]), v["k"]).tolist() == v["perms"]
    for v in vec["stable_sort_permutation"]:
        assert oracle.piecewise_sort(np.array(v["x"]), len(v["x"])).tolist()[0] == v["perm"]
    for v in vec["window_spec"]:
        st, h, b, _ = oracle.window_spec(v["n"], v["k"])
        if "error" in v:
            assert st == 3
        else:
            assert (st, h, b) == (0, v["h"], v["b"])


def test_golden_small_cases(oracle):
    z = np.load(os.path.join(GOLDEN, "small_cases.npz"))
    n = len([f for f in z.files if f.endswith("_x")])
    for i in range(n):
        x, k, y = z[f"c{i}_x"], int(z[f"c{i}_k"]), z[f"c{i}_y"]
        assert same(oracle.median_filter(x, k), y), f"case {i} k={k} {x.dtype}"


def test_exhaustive_small_alphabet(oracle):
    """verify.hpp:142-158: every vector of length <= 8 over {0,1,2}, every odd k <= n."""
    cases = 0
    for n in range(1, 9):
        for tup in itertools.product(range(3), repeat=n):
            x = np.array(tup, dtype=np.int64)
            for k in range(1, n + 1, 2):
                assert np.array_equal(oracle.median_filter(x, k), oracle.naive(x, k)), (tup, k)
                cases += 1
    assert cases > 30000


def test_state_invariants(oracle):
    """Eq. 4 on kept windows: s_A + s_B = h before every emit."""
    rng = np.random.default_rng(7)
    for k in (3, 7, 31, 101):
        for n in (5 * k, 5 * k + 3):
            x = rng.integers(0, 6, size=n)
            y, tr = oracle.median_filter_trace(x, k)
            h = (k - 1) // 2
            steps = tr[1:]  # entry 0 is the construct peek
            assert np.all(steps[:, 2] + steps[:, 3] == h)
            assert np.array_equal(y, oracle.naive(x, k))


def test_against_reference_random(oracle, reference):
    rng = np.random.default_rng(42)
    for k in (1, 3, 5, 31, 101, 255, 1023, 2049):
        for dt in (np.int32, np.int64, np.float32, np.float64):
            for _ in range(3):
                n = int(rng.integers(1, 6 * k + 50))
                if dt in (np.float32, np.float64):
                    x = rng.standard_normal(n).astype(dt)
                else:
                    x = rng.integers(-20, 20, size=n).astype(dt)
                assert same(oracle.median_filter(x, k), reference.median_filter(x, k)), (k, dt, n)


def test_reference_run_verify(reference):
    ok, exhaustive, rnd = reference.run_verify(6, 50, 0)
    assert ok and exhaustive > 0 and rnd == 50
    ok, _, _ = reference.run_verify(5, 10, 0, inject_fault=True)
    assert not ok  # the harness catches the deliberately broken filter (verify.hpp:40-52)


def test_piecewise_sort_vs_reference(oracle, reference):
    rng = np.random.default_rng(3)
    for k in (1, 3, 31, 255, 1025):
        x = rng.integers(0, 5, size=4 * k + 7)
        assert np.array_equal(oracle.piecewise_sort(x, k), reference.piecewise_sort(x, k))


def test_generators_vs_reference(oracle, reference):
    for kind in range(7):
        for width in (32, 64):
            assert np.array_equal(oracle.generate(kind, 5000, 11, width), reference.generate(kind, 5000, 11, width))


def test_config_input_checksums(oracle):
    """The SURVEY.md §8(d) recipes reproduce the golden input checksums (small configs)."""
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))
    assert oracle.fold_checksum(oracle.uniform_f64(1, 1_000_000)) == cfg["c1"]["in_cksum"]
    assert oracle.fold_checksum(oracle.uniform_f32(2, 1 << 26)) == cfg["c2_k3"]["in_cksum"]


def test_config1_output(oracle):
    cfg = json.load(open(os.path.join(GOLDEN, "configs.json")))["c1"]
    y = oracle.median_filter(oracle.uniform_f64(1, 1_000_000), 101)
    assert y.size == cfg["out_len"] and oracle.fold_checksum(y) == cfg["out_cksum"]


def test_keymap_is_involution_and_monotone():
    rng = np.random.default_rng(1)
    b = rng.integers(0, 2**32, size=10000, dtype=np.uint64).astype(np.uint32).view(np.float32)
    k = keymap(b)
    assert np.array_equal(unkey(k, np.float32).view(np.int32), b.view(np.int32))
    f = np.array([-np.inf, -1.0, -0.0, 0.0, 1e-30, 1.0, np.inf], dtype=np.float32)
    assert np.all(np.diff(keymap(f).astype(np.int64)) > 0)


def test_shard_identity_oracle(oracle):
    """Halo sharding reproduces the unsharded output."""
    import paper_1406_1717_b200.shard as sh
    rng = np.random.default_rng(9)
    for k in (3, 31, 255):
        x = rng.integers(0, 9, size=40 * k + 5)
        whole = oracle.median_filter(x, k)
        for world in (2, 3, 8):
            parts = [sh.run_shard(x, k, s, oracle.median_filter) for s in sh.shard_outputs(x.size, k, world)]
            assert np.array_equal(np.concatenate(parts), whole)
        assert np.array_equal(oracle.median_filter_threads(x, k, 4), whole)
