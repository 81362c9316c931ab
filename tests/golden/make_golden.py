"""Regenerate the committed golden fixtures from the REFERENCE itself.

Run in the build container (needs oracle/_ref/libmedfilt_ref.so, i.e. the unmodified
reference headers compiled by oracle/Makefile):

    python tests/golden/make_golden.py            # small fixtures + configs.json
    python tests/golden/make_golden.py --configs  # also recompute the five BASELINE configs (~3 min)

Outputs (committed; nothing reads /root/reference at test time):
  small_cases.npz  -- seeded small signals across dtypes / k / value distributions with
                      the reference's median_filter output (floats through the key map)
  spec_vectors.json -- SPEC.md known answers, each re-derived by the reference
  configs.json     -- in/out fold_checksum (io.hpp:17-28) of the five BASELINE configs
                      (inputs: SURVEY.md §8(d) recipe; outputs: reference median_filter,
                      8-way halo-sharded, shard-identity proven in tests/test_oracle.py)
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_lib import Oracle, Reference, keymap, unkey  # noqa: E402


def small_cases(ref: Reference, orc: Oracle):
    rng = np.random.default_rng(20261019)
    cases = {}
    ks = [1, 3, 5, 7, 9, 15, 31, 33, 63, 101, 127, 255, 257, 511, 1023, 1025, 2049, 4097]
    idx = 0
    for k in ks:
        for dt in (np.int32, np.int64, np.float32, np.float64):
            for dist in ("wide", "ties", "sorted", "special"):
                n = int(rng.integers(max(1, k - 2), 3 * k + 70))
                if dist == "wide":
                    if dt in (np.int32, np.int64):
                        info = np.iinfo(dt)
                        x = rng.integers(info.min, info.max, size=n, dtype=dt, endpoint=True)
                    else:
                        x = rng.standard_normal(n).astype(dt) * dt(1e3)
                elif dist == "ties":
                    x = rng.integers(0, 4, size=n).astype(dt)
                elif dist == "sorted":
                    x = np.sort(rng.integers(-50, 50, size=n)).astype(dt)
                    if rng.integers(2):
                        x = x[::-1].copy()
                else:
                    if dt in (np.int32, np.int64):
                        info = np.iinfo(dt)
                        pool = np.array([info.min, info.max, 0, -1, 1, info.max - 1, info.min + 1], dtype=dt)
                    else:
                        bits = np.dtype(dt).itemsize * 8
                        ui = np.uint32 if bits == 32 else np.uint64
                        nan_pay = np.array([0x7FC00001, 0xFFC00002] if bits == 32 else
                                           [0x7FF8000000000001, 0xFFF8000000000002], dtype=ui).view(dt)
                        pool = np.concatenate([np.array([0.0, -0.0, np.inf, -np.inf, 1.5, -1.5,
                                                         np.finfo(dt).max, -np.finfo(dt).tiny], dtype=dt),
                                               nan_pay])
                    x = pool[rng.integers(0, pool.size, size=n)]
                y = ref.median_filter(x, k)
                cases[f"c{idx}_x"] = x
                cases[f"c{idx}_k"] = np.array(k)
                cases[f"c{idx}_y"] = y
                idx += 1
    np.savez_compressed(os.path.join(HERE, "small_cases.npz"), **cases)
    print("small cases:", idx)


def spec_vectors(ref: Reference):
    # Known answers quoted by the reference's SPEC.md (line numbers given), each also
    # re-derived here by running the reference.
    vec = {
        "median_filter": [
            {"x": [5, 1, 3, 2, 4], "k": 3, "y": [3, 2, 3]},
            {"x": [1, 5, 2, 8, 3, 9, 4], "k": 7, "y": [4]},
            {"x": [2, 1], "k": 3, "y": []},
            {"x": [1, 2, 3, 4, 5, 6], "k": 1, "y": [1, 2, 3, 4, 5, 6]},
            {"x": [7, 7, 7, 7, 7], "k": 3, "y": [7, 7, 7]},
        ],
        "piecewise_sort": [
            {"x": [5, 1, 3, 2, 4, 6], "k": 3, "perms": [[1, 2, 0], [0, 1, 2]]},
            {"x": [6, 5, 4, 3, 2, 1], "k": 3, "perms": [[2, 1, 0], [2, 1, 0]]},
            {"x": [4, 4, 4, 4, 4, 4], "k": 3, "perms": [[0, 1, 2], [0, 1, 2]]},
        ],
        "stable_sort_permutation": [  # SPEC.md:67-69 (one block: k = len)
            {"x": [3, 1, 3], "perm": [1, 0, 2]},
            {"x": [1, 2, 3], "perm": [0, 1, 2]},
            {"x": [7, 7, 7], "perm": [0, 1, 2]},
        ],
        "window_spec": [
            {"n": 6, "k": 3, "h": 1, "b": 2},
            {"n": 5, "k": 3, "h": 1, "b": 2},
            {"n": 4, "k": 4, "error": "even window size unsupported (window must be k = 2h+1)"},
        ],
        "sort_via_median_filter": [
            {"blocks": [[4, 2]], "sorted": [[2, 4]]},
            {"blocks": [[1, 2, 3]], "sorted": [[1, 2, 3]]},
            {"blocks": [[3, 1], [9, 7]], "sorted": [[1, 3], [7, 9]]},
        ],
    }
    for v in vec["median_filter"]:
        got = ref.median_filter(np.array(v["x"], dtype=np.int64), v["k"]).tolist()
        assert got == v["y"], (v, got)
    for v in vec["piecewise_sort"]:
        got = ref.piecewise_sort(np.array(v["x"]), v["k"]).tolist()
        assert got == v["perms"], (v, got)
    for v in vec["stable_sort_permutation"]:
        got = ref.piecewise_sort(np.array(v["x"]), len(v["x"])).tolist()[0]
        assert got == v["perm"], (v, got)
    for v in vec["sort_via_median_filter"]:
        got = ref.sort_via_median_filter(np.array(v["blocks"])).tolist()
        assert got == v["sorted"], (v, got)
    with open(os.path.join(HERE, "spec_vectors.json"), "w") as f:
        json.dump(vec, f, indent=1)
    print("spec vectors verified against the reference")


def configs(ref: Reference, orc: Oracle):
    res = {}

    def rec(name, x, k, y, extra=None):
        d = dict(k=k, in_len=int(x.size), in_cksum=orc.fold_checksum(x), out_len=int(y.size),
                 out_cksum=orc.fold_checksum(y), y0_key=int(keymap(y.ravel()[:1])[0]),
                 ylast_key=int(keymap(y.ravel()[-1:])[0]))
        d.update(extra or {})
        res[name] = d
        print(name, d, flush=True)

    x = orc.uniform_f64(1, 1_000_000)
    rec("c1", x, 101, ref.median_filter(x, 101))
    x = orc.uniform_f32(2, 1 << 26)
    for k in (3, 31, 255, 1023):
        rec(f"c2_k{k}", x, k, unkey(ref.median_filter_threads(keymap(x), k, 8), np.float32))
    x = orc.mod_i32(3, 16, 4096 * 65536).reshape(4096, 65536)
    y = ref.median_filter_rows(x, 255, 8)
    rec("c3", x.ravel(), 255, y.ravel(), {"rows": 4096, "row_len": 65536,
                                           "row0_out_cksum": orc.fold_checksum(y[0].copy())})
    x = orc.trend_f64(4, 1 << 27)
    rec("c4", x, 10001, unkey(ref.median_filter_threads(keymap(x), 10001, 8), np.float64))
    del x
    x = orc.uniform_f32(5, 1 << 30)
    rec("c5", x, 100001, unkey(ref.median_filter_threads(keymap(x), 100001, 8), np.float32))
    with open(os.path.join(HERE, "configs.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    ref, orc = Reference(), Oracle()
    small_cases(ref, orc)
    spec_vectors(ref)
    if "--configs" in sys.argv:
        configs(ref, orc)
