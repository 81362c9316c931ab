"""GPU checks of the multi-device and multi-stream paths (SURVEY.md §8(b) "Multi-GPU entry:
a device list", §8(e)).

The box has one GPU, so the multi-device context is driven over the device listed twice:
that runs the real sharding, the per-device host threads and the D2H-at-offset gather
(two sub-contexts with their own streams on one GPU).  It is a correctness test, never a
timing.  The bench's multi-rank path is driven by torchrun with two gloo ranks sharing
the GPU, and its chained fold_checksum must equal one device filtering the global signal.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1406_1717_b200 as mf
from paper_1406_1717_b200 import _native as N

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def bits(a):
    a = np.ascontiguousarray(a)
    return a.view(np.int32 if a.itemsize == 4 else np.int64)


@pytest.fixture(scope="module")
def multi():
    return mf.Context.multi([0, 0])


def test_multi_context_devices(multi):
    assert multi.devices == [0, 0]
    assert mf.Context.get(0).devices == [0]


@pytest.mark.parametrize("dt", (np.float32, np.int64), ids=lambda d: np.dtype(d).name)
@pytest.mark.parametrize("k", [3, 31, 255, 1023, 4097])
def test_multi_device_signal_equals_single(multi, dt, k):
    """A signal big enough to split (>= 2 x 2^20 outputs per shard): the halo'd shards
    of the two devices land at their offsets of one host output."""
    rng = np.random.default_rng(k)
    n = (3 << 20) + 12345
    x = (rng.standard_normal(n) * 100).astype(dt)
    want = mf.median_filter(x, k, ctx=mf.Context.get(0))
    got = mf.median_filter(x, k, ctx=multi)
    assert np.array_equal(bits(got), bits(want))
    assert multi.last_launches() >= 2          # both devices launched


@pytest.mark.parametrize("k", [31, 255, 2049])
def test_multi_device_rows_equal_single(multi, oracle, k):
    rng = np.random.default_rng(7)
    x = rng.integers(0, 16, size=(9, 3 * k + 17)).astype(np.int32)
    got = mf.median_filter_rows(x, k, ctx=multi)
    want = np.stack([oracle.median_filter(r, k) for r in x])
    assert np.array_equal(got, want)


def test_multi_device_small_signal_and_errors(multi, oracle):
    x = np.arange(1000, dtype=np.int32)[::-1].copy()
    assert np.array_equal(mf.median_filter(x, 31, ctx=multi), oracle.median_filter(x, 31))
    assert mf.median_filter(x[:5], 7, ctx=multi).size == 0
    with pytest.raises(mf.InvalidArgument, match="^even window size"):
        mf.median_filter(x, 4, ctx=multi)
    # host memory through a device entry is refused
    L = N.lib()
    y = np.empty(x.size, dtype=x.dtype)
    assert L.mf_median_filter_device(multi.handle, N.MF_I32, C.c_void_p(x.ctypes.data), x.size, 31,
                                     C.c_void_p(y.ctypes.data), None) == N.MF_BAD_ARG


def test_cpp_set_devices_multi():
    """gpu.hpp's set_devices({0, 0}) -> the FilterFn-shaped median_filter shards."""
    exe = os.path.join(ROOT, "tests", "cpp", "_bin", "gpu_multi_check")
    if not os.path.exists(exe):
        pytest.skip("tests/cpp not built")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300,
                       env=dict(os.environ, MEDFILT_GPU_DEVICES="0,0"))
    assert r.returncode == 0, r.stdout + r.stderr


def test_workspace_ordered_across_streams(oracle):
    """Two large-k calls on one context issued on two streams: the shared workspace is
    ordered by the context's event, so neither corrupts the other."""
    import torch
    ctx = mf.Context(0)
    rng = np.random.default_rng(3)
    k = 4097
    xs = [rng.standard_normal(40 * k + 11).astype(np.float32) for _ in range(2)]
    wants = [oracle.median_filter(x, k) for x in xs]
    ss = [torch.cuda.Stream(), torch.cuda.Stream()]
    xd = [torch.from_numpy(x).cuda() for x in xs]
    torch.cuda.synchronize()
    for _ in range(3):
        outs = []
        for x, s in zip(xd, ss):
            with torch.cuda.stream(s):
                outs.append(mf.median_filter_device(x, k, stream=s, ctx=ctx))
        torch.cuda.synchronize()
        for o, w in zip(outs, wants):
            assert np.array_equal(bits(o.cpu().numpy()), bits(w))


def test_large_class_rejects_k_past_limit():
    """k > 2^31 - 65 in the large class: MF_BAD_ARG before any device work (the pipeline
    packs 2k positions into 32 bits); the reference's own limit, k < 2^32 - 1, is
    MF_K_TOO_LARGE."""
    L = N.lib()
    ctx = mf.Context(0)
    k = (1 << 31) + 1
    fake = C.c_void_p(0x1000)
    st = L.mf_median_filter_device(ctx.handle, N.MF_F32, fake, k + 10, k, fake, None)
    assert st == N.MF_BAD_ARG
    k_ok = (1 << 31) - 65
    assert L.mf_window_spec(k_ok, k_ok, None, None, None) == N.MF_OK


def test_bench_two_ranks_gloo_match_single_device():
    """bench.py under torchrun with two gloo ranks sharing the GPU (a functional check of
    the N > 1 path, not a timing): every k's chained fold_checksum of the concatenated
    rank outputs equals one device filtering the same global signal."""
    import torch
    n = 1 << 22
    env = dict(os.environ, MF_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29611", os.path.join(ROOT, "bench.py"),
           "--gpus", "2", "--steps", "2", "--warmup", "3", "--n-per-gpu", str(n), "--no-cpu"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2
    x = mf.generate_device("uniform_f32", 2, 2 * n)
    for k in (3, 31, 255, 1023):
        y = mf.median_filter_device(x, k).cpu().numpy()
        assert int(line["checksums"][str(k)]["out_cksum"]) == mf.fold_checksum(y), k
    # the gathered output of the dominant k is the whole global output, not more
    kg = line["gather"]["k"]
    assert line["gather"]["bytes"] == (2 * n - kg + 1) * 4
    torch.cuda.synchronize()


@pytest.mark.parametrize("k", [31, 45, 255, 1023, 2049])
def test_repeat_determinism_under_concurrency(oracle, k):
    """Race smoke test (compute-sanitizer is closed on the pool): the same filter issued 12
    times over four streams with four contexts, so CTAs of different launches share SMs and
    schedules vary; every result must be bit-identical to the oracle's."""
    import torch
    rng = np.random.default_rng(77 + k)
    x = (rng.standard_normal(400_003) * 10).astype(np.float32)
    x[rng.integers(0, x.size, 4000)] = 1.5            # some ties
    want = bits(oracle.median_filter(x, k))
    xd = torch.from_numpy(x).cuda()
    ctxs = [mf.Context(0) for _ in range(4)]
    ss = [torch.cuda.Stream() for _ in range(4)]
    outs = []
    for rep in range(12):
        s = ss[rep % 4]
        with torch.cuda.stream(s):
            outs.append(mf.median_filter_device(xd, k, stream=s, ctx=ctxs[rep % 4]))
    torch.cuda.synchronize()
    for rep, o in enumerate(outs):
        assert np.array_equal(bits(o.cpu().numpy()), want), f"k={k} repetition {rep}"


def test_multi_device_shard_counts(multi, oracle):
    """Fewer rows than devices, one row, and signals just above and below the minimum
    shard size all give the single-device result."""
    rng = np.random.default_rng(12)
    xr = rng.integers(-9, 9, size=(1, 5000)).astype(np.int64)
    assert np.array_equal(mf.median_filter_rows(xr, 101, ctx=multi)[0], oracle.median_filter(xr[0], 101))
    for n in ((1 << 21) + 100 - 1, (1 << 21) + 300):     # keep below / above 2 x 2^20 outputs
        x = rng.standard_normal(n).astype(np.float32)
        assert np.array_equal(bits(mf.median_filter(x, 201, ctx=multi)),
                              bits(mf.median_filter(x, 201, ctx=mf.Context.get(0))))


@pytest.mark.parametrize("k", [3, 31, 255, 1023, 4097])
def test_multi_device_device_pointers_equal_single(multi, k):
    """Device-resident input on the multi-device context: shards copied peer to peer (the
    second listed device copies even when it is the same GPU), filtered on each device and
    copied back to their offsets, stream-ordered on the caller's stream."""
    import torch
    x = mf.generate_device("uniform_f32", 31, (3 << 20) + 77)
    want = mf.median_filter_device(x, k).cpu().numpy()
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        got = mf.median_filter_device(x, k, ctx=multi, stream=s)
    s.synchronize()
    assert np.array_equal(bits(got.cpu().numpy()), bits(want))


def test_multi_device_device_rows_strided():
    """Rows on device with row strides wider than the rows: row groups go to the devices
    and the outputs' row gaps are left untouched."""
    import torch
    multi = mf.Context.multi([0, 0, 0])
    xr = mf.generate_device("mod_i32", 5, 7 * 30_011, mod=16).view(7, 30_011)
    big = torch.zeros((7, 30_011 + 5), dtype=torch.int32, device="cuda")
    big[:, :30_011] = xr
    keep = 30_011 - 255 + 1
    out = torch.full((7, keep + 9), -1, dtype=torch.int32, device="cuda")
    L = N.lib()
    assert L.mf_median_filter_rows_device(multi.handle, N.MF_I32, C.c_void_p(big.data_ptr()), 7, 30_011,
                                          30_011 + 5, 255, C.c_void_p(out.data_ptr()), keep + 9, None) == 0
    torch.cuda.synchronize()
    want = mf.median_filter_rows_device(xr, 255).cpu().numpy()
    o = out.cpu().numpy()
    assert np.array_equal(o[:, :keep], want)
    assert (o[:, keep:] == -1).all()
