#!/usr/bin/env python3
"""Benchmark of the B200 median-filter hot path (BASELINE.json metric).

Metric: median-filter output samples/s (whole job, all ranks) and the fraction of the
HBM roofline.  Default workload = BASELINE config 2: a float32 signal of 2^26 samples
per GPU (SplitMix64 seed 2 uniform[0,1)) filtered at every k of the
sweep {3, 31, 255, 1023}; one step = the whole sweep (four filter calls).  Inputs
(268 MB per GPU) exceed the 126 MB L2, so no flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2|c1|c3|c4|c5] [--impl ours|reference]

N > 1 (torchrun, one rank per GPU): weak scaling.  The global signal has N * 2^26
samples; rank g filters its contiguous output range with a (k-1)-sample halo
(paper_1406_1717_b200.shard), generated in place on its own GPU.  No collective
touches the data path; the timing barrier and max-over-ranks reduction are the only
NCCL calls.

--impl reference times the reference's own CPU implementation (oracle/_ref: the
unmodified reference headers, halo-sharded over every host core) on the same
config/metric; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (dtype, n_per_gpu, ks, generator, seed, rows)
    "c1": ("float64", 1_000_000, (101,), "uniform_f64", 1, 1),
    "c2": ("float32", 1 << 26, (3, 31, 255, 1023), "uniform_f32", 2, 1),
    "c3": ("int32", 65536, (255,), "mod_i32", 3, 4096),
    "c4": ("float64", 1 << 27, (10001,), "trend_f64", 4, 1),
    "c5": ("float32", 1 << 30, (100001,), "uniform_f32", 5, 1),
}
WORKLOAD = {
    "c1": "config1: n=1e6 f64 uniform seed1, k=101",
    "c2": "config2: n=2^26 f32 uniform seed2 per GPU, k sweep {3,31,255,1023} (one step = all four)",
    "c3": "config3: 4096 rows x 65536 i32 uniform[0,16) seed3, k=255",
    "c4": "config4: n=2^27 f64 i/n+N(0,0.01) seed4, k=10001",
    "c5": "config5: n=2^30 f32 uniform seed5, k=100001",
}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        if not self.rows:
            return None
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def input_range(cfg, rank, world):
    """[begin, end) of the global signal this rank needs: the union over every k of its
    halo'd shard (paper_1406_1717_b200.shard.input_union).  Pure arithmetic, CPU-tested."""
    from paper_1406_1717_b200.shard import input_union
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    return input_union(n * world, ks, world, rank)


def make_input(cfg, rank, world, device):
    """This rank's input slice of the global signal (device resident) and its begin."""
    import torch
    import paper_1406_1717_b200 as mf
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    if rows > 1:   # batched rows: shard whole rows, global row r = stream offset r*n
        r0, r1 = mf.shard_rows(rows * world, world)[rank]
        x = mf.generate_device(gen, seed, (r1 - r0) * n, offset=r0 * n, device=device, mod=16)
        return x.view(r1 - r0, n), r0
    begin, end = input_range(cfg, rank, world)
    if gen == "trend_f64":
        full = mf.generate_trend_f64(seed, end)
        return torch.from_numpy(full[begin:end]).to(f"cuda:{device}"), begin
    return mf.generate_device(gen, seed, end - begin, offset=begin, device=device), begin


def shard_views(cfg, x, begin, rank, world, k):
    """(input view, n_out) of this rank's shard for window k; the view always holds the
    shard's n_in samples (shard_view raises otherwise)."""
    from paper_1406_1717_b200.shard import shard_outputs, shard_view
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    sh = shard_outputs(n * world, k, world)[rank]
    return shard_view(x, begin, sh), sh.n_out


def golden(cfg, k):
    """Reference fold_checksum of the config's full output (tests/golden/configs.json,
    produced by the reference itself)."""
    p = os.path.join(ROOT, "tests", "golden", "configs.json")
    if not os.path.exists(p):
        return None
    g = json.load(open(p))
    return g.get(f"{cfg}_k{k}", g.get(cfg))


def output_checksums(cfg, jobs, outs, world, rank, dist):
    """fold_checksum (io.hpp:17-28) of every k's global output, chained over ranks in
    rank order, and (N = 1) the reference's golden value for the same config."""
    import paper_1406_1717_b200 as mf
    from paper_1406_1717_b200.shard import chained_fold_checksum
    res = {}
    for k, xv, nout in jobs:
        y = outs[k]
        y = (y[:, :xv.shape[1] - k + 1] if y.dim() == 2 else y[:nout]).contiguous().cpu().numpy()
        h = chained_fold_checksum(y, world, rank, dist=dist if world > 1 else None, fold=mf.fold_checksum)
        if rank == 0:
            ent = {"out_cksum": str(h)}
            gd = golden(cfg, k)
            if world == 1 and gd is not None and gd.get("k") == k:
                ent["golden"] = str(gd["out_cksum"])
                ent["match"] = h == gd["out_cksum"]
            res[str(k)] = ent
    return res


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_1406_1717_b200 as mf

    world, rank, local = dist_env()
    # one rank per GPU; MF_BENCH_BACKEND=gloo lets several ranks share a GPU for a smoke test
    backend = os.environ.get("MF_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        else:
            dist.init_process_group(backend)
    red_dev = f"cuda:{local}" if backend == "nccl" else "cpu"
    cfg = args.config
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    ctx = mf.Context.get(local)
    stream = torch.cuda.Stream(device=local)
    width = np.dtype(dtype).itemsize

    with torch.cuda.stream(stream):
        if rows > 1:
            x, _r0 = make_input(cfg, rank, world, local)
            jobs = [(k, x, x.shape[0] * (n - k + 1)) for k in ks]
            outs = {k: torch.empty((x.shape[0], n - k + 1), dtype=x.dtype, device=x.device) for k in ks}
        else:
            x, begin = make_input(cfg, rank, world, local)
            jobs = []
            outs = {}
            for k in ks:
                xv, n_out = shard_views(cfg, x, begin, rank, world, k)
                jobs.append((k, xv, n_out))
                outs[k] = torch.empty(max(n_out, 1), dtype=x.dtype, device=x.device)
    stream.synchronize()

    def call(k, xv):
        if rows > 1:
            mf.median_filter_rows_device(xv, k, out=outs[k], stream=stream, ctx=ctx)
        else:
            mf.median_filter_device(xv, k, out=outs[k], stream=stream, ctx=ctx)
        return ctx.last_launches()

    # per-k event pairs for the kernel share / roofline
    ev = {k: [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
              for _ in range(args.steps)] for k in ks}
    for _ in range(args.warmup):
        for k, xv, _n in jobs:
            call(k, xv)
    stream.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    launches = 0
    t0.record(stream)
    for s in range(args.steps):
        for k, xv, _n in jobs:
            ev[k][s][0].record(stream)
            launches += call(k, xv)
            ev[k][s][1].record(stream)
    t1.record(stream)
    stream.synchronize()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clock = clocks.stop()
    ms = t0.elapsed_time(t1)
    per_k_ms = {k: statistics.mean(a.elapsed_time(b) for a, b in ev[k]) for k in ks}
    outputs_rank = sum(nout for _k, _x, nout in jobs)
    if world > 1:  # per-k kernel times: max over ranks, so every rank picks the same dominant k
        pk = torch.tensor([per_k_ms[k] for k in ks], dtype=torch.float64, device=red_dev)
        dist.all_reduce(pk, op=dist.ReduceOp.MAX)
        per_k_ms = {k: float(v) for k, v in zip(ks, pk.tolist())}
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        o = torch.tensor([outputs_rank], dtype=torch.float64, device=red_dev)
        dist.all_reduce(o, op=dist.ReduceOp.SUM)
        outputs_total = float(o.item())
    else:
        outputs_total = float(outputs_rank)
    ms_per_step = ms / args.steps
    value = outputs_total * args.steps / (ms / 1e3)

    # roofline of the dominant kernel (largest time share of the step)
    peak, peak_src = load_peaks()
    kdom = max(per_k_ms, key=per_k_ms.get)
    kk, xv, nout = [j for j in jobs if j[0] == kdom][0]
    alg_bytes = (xv.numel() + nout) * width
    achieved = alg_bytes / (per_k_ms[kdom] / 1e3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get(f"{cfg}_k{kdom}")

    # per-phase device times of one extra (untimed) call per k (MF_OPT_PROFILE events)
    phases = None
    if rank == 0 and not args.no_check:
        ctx.profile(True)
        phases = {}
        for k, xv, _n in jobs:
            call(k, xv)
            phases[str(k)] = [[name, ms] for name, ms in ctx.last_phases()]
        ctx.profile(False)

    # fold_checksum of every k's global output (chained over ranks), against the golden
    checks = None
    if not args.no_check:
        checks = output_checksums(cfg, jobs, outs, world, rank, dist)

    # optional final gather of the dominant k's outputs onto rank 0 (device gather over
    # NCCL; reported separately, outside the timed region)
    gather = None
    if world > 1 and not args.no_gather:
        from paper_1406_1717_b200.shard import gather_outputs_device
        kk0, xv0, nout0 = [j for j in jobs if j[0] == max(per_k_ms, key=per_k_ms.get)][0]
        part = outs[kk0][:nout0] if rows == 1 else outs[kk0]
        if backend != "nccl":
            part = part.cpu()
        dist.barrier()
        g0 = time.perf_counter()
        full = gather_outputs_device(part, world, rank, dist=dist)
        if full is not None and full.is_cuda:
            torch.cuda.synchronize()
        gms = (time.perf_counter() - g0) * 1e3
        if rank == 0:
            gather = {"k": kk0, "ms": gms, "bytes": int(full.numel() * full.element_size()),
                      "how": "torch.distributed.gather of padded device tensors (NCCL send/recv)" if backend == "nccl"
                             else "torch.distributed.gather (gloo, host tensors)"}
        del full

    # end to end through the public host API (host buffers, H2D + D2H timed), every rank
    # on its own shard, max over ranks
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(cfg, jobs, args, width, world, dist, red_dev)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(cfg, args)

    if rank == 0:
        line = {
            "metric": "median-filter output samples/sec",
            "value": value,
            "unit": "samples/s",
            "n_gpus": world,
            "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms_per_step,
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": {"float32": "f32", "float64": "f64", "int32": "i32"}[dtype],
            "data": "synthetic: SplitMix64 (generators.hpp:16-29) recipe of SURVEY.md §8(d), generated on device",
            "config": {"workload": WORKLOAD[cfg], "n_per_gpu": n * rows, "k": list(ks),
                       "parallelism": f"halo-sharded outputs x{world}" if rows == 1 else f"rows x{world}",
                       "l2": "inputs exceed L2 (no flush needed)" if n * rows * width > 126e6 else
                             "input fits L2 (warm)",
                       "per_k_ms": {str(k): per_k_ms[k] for k in ks},
                       "per_k_samples_per_s": {str(k): [j[2] for j in jobs if j[0] == k][0] * world / (per_k_ms[k] / 1e3)
                                               for k in ks}},
            "checksums": checks,
            "phases": phases,
            "gather": gather,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel_k": kdom,
                         "algorithmic_bytes_per_launch": alg_bytes, "peak_source": peak_src},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clock,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(cfg, jobs, args, width, world=1, dist=None, red_dev="cpu"):
    """Same metric through the host-buffer C ABI (mf_median_filter / _rows, the literal
    drop-in): every step copies the input H2D and the medians D2H inside the timed region.
    Measured twice: from pinned host buffers (the headline) and from pageable ones (what a
    std::vector caller of gpu.hpp hands over).  Every rank runs its own shard; the time is
    the max over ranks and the value counts all ranks' outputs."""
    import torch
    import paper_1406_1717_b200 as mf
    import ctypes as C
    from paper_1406_1717_b200 import _native as N
    from paper_1406_1717_b200.filter import _DTYPES, _check
    ctx = mf.Context.get(torch.cuda.current_device())
    L = N.lib()
    steps = max(1, min(args.steps, 5))
    outputs = sum(n for _k, _x, n in jobs)
    res = {}
    for mode in ("pinned", "pageable"):
        hx, hy = {}, {}
        for k, xv, nout in jobs:
            shape = (xv.shape[0], xv.shape[1] - k + 1) if xv.dim() == 2 else (max(nout, 1),)
            if mode == "pinned":
                hx[k] = xv.cpu().pin_memory().numpy()
                hy[k] = torch.empty(shape, dtype=xv.dtype).pin_memory().numpy()
            else:
                hx[k] = xv.cpu().numpy().copy()
                hy[k] = np.empty(shape, dtype=hx[k].dtype)

        def one(k):
            x, y = hx[k], hy[k]
            if x.ndim == 2:
                _check(L.mf_median_filter_rows(ctx.handle, _DTYPES[x.dtype], x.ctypes.data, x.shape[0], x.shape[1],
                                               x.shape[1], k, y.ctypes.data, y.shape[1]))
            else:
                ylen = C.c_size_t()
                _check(L.mf_median_filter(ctx.handle, _DTYPES[x.dtype], x.ctypes.data, x.size, k, y.ctypes.data,
                                          y.size, C.byref(ylen)))
        for k, _x, _n in jobs:
            one(k)
        if world > 1:
            dist.barrier()
        t = time.perf_counter()
        for _ in range(steps):
            for k, _x, _n in jobs:
                one(k)
        dt = time.perf_counter() - t
        tot = outputs
        if world > 1:
            tt = torch.tensor([dt], dtype=torch.float64, device=red_dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            dt = float(tt.item())
            o = torch.tensor([float(outputs)], dtype=torch.float64, device=red_dev)
            dist.all_reduce(o, op=dist.ReduceOp.SUM)
            tot = float(o.item())
        res[mode] = {"value": tot * steps / dt, "steps": steps,
                     "h2d_bytes_per_step": int(sum(hx[k].nbytes for k in hx)),
                     "d2h_bytes_per_step": int(sum(hy[k].nbytes for k in hy))}
        del hx, hy
    p = res["pinned"]
    return {"value": p["value"], "unit": "samples/s", "h2d_bytes_per_step": p["h2d_bytes_per_step"],
            "d2h_bytes_per_step": p["d2h_bytes_per_step"], "steps": p["steps"],
            "api": "mf_median_filter / mf_median_filter_rows (host buffers, pinned); per-rank bytes",
            "pageable_value": res["pageable"]["value"]}


def _ref_lib():
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Reference, Oracle  # noqa: E402  (the checker/baseline leg only)
    if Reference.available():
        return Reference(), "reference"
    return Oracle(), "port"


def _host_input(cfg, n_sample):
    """The config's input on the host (same bits as the device generator)."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    from oracle_lib import Oracle
    o = Oracle()
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    if gen == "uniform_f32":
        return o.uniform_f32(seed, n_sample)
    if gen == "uniform_f64":
        return o.uniform_f64(seed, n_sample)
    if gen == "mod_i32":
        return o.mod_i32(seed, 16, n_sample)
    return o.trend_f64(seed, n_sample)


def _keyed_input(lib, kind, cfg, n_sample):
    """The config's input on the host, already key-mapped (floats -> signed totalOrder
    keys) and in the width the reference instantiation takes: the key
    map is not part of the timed reference path."""
    from oracle_lib import keymap
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    kx = np.ascontiguousarray(keymap(_host_input(cfg, n_sample)))
    if kind != "reference":
        kx = kx.astype(np.int64)
    return kx.reshape(-1, n) if rows > 1 else kx


def _time_ref(lib, kind, cfg, kx, threads):
    """One pass of the reference over the keyed input (every k of the config): the
    reference's median_filter<T> halo-sharded over `threads` host threads, or rows over
    threads.  Returns (outputs, seconds)."""
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    outs = 0
    t = time.perf_counter()
    for k in ks:
        if rows > 1:
            if kind == "reference":
                lib.median_filter_rows(kx, k, threads)
            else:
                for r in range(kx.shape[0]):
                    lib.median_filter_threads(kx[r], k, threads)
            outs += kx.shape[0] * (n - k + 1)
        else:
            lib.median_filter_threads(kx, k, threads)
            outs += kx.size - k + 1
    return outs, time.perf_counter() - t


def _sample(cfg, cap):
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    sample = min(n * rows, cap)
    if rows > 1:
        sample = max(n, sample // n * n)
    return sample


def _sample_text(cfg, sample, threads):
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    whole = "the whole" if sample >= n * rows else f"the first {sample} samples of the"
    return (f"{whole} {cfg} signal ({sample} samples{f', {sample // n} rows' if rows > 1 else ''}), every k of "
            f"the config, input key-mapped before timing, {'rows' if rows > 1 else 'halo-sharded'} over "
            f"{threads} host threads")


def cpu_baseline(cfg, args):
    """The reference CPU path on this host (all threads) on a bounded sample of the same
    workload: 1 warm-up, 3 repeats, median (bench.hpp:100-122)."""
    lib, kind = _ref_lib()
    threads = os.cpu_count() or 1
    sample = _sample(cfg, args.cpu_sample)
    kx = _keyed_input(lib, kind, cfg, sample)
    _time_ref(lib, kind, cfg, kx, threads)
    runs = [_time_ref(lib, kind, cfg, kx, threads) for _ in range(3)]
    outs = runs[0][0]
    dt = statistics.median(r[1] for r in runs)
    return {"value": outs / dt, "unit": "samples/s", "cores": threads, "kind": kind,
            "sample": _sample_text(cfg, sample, threads) + "; median of 3 after 1 warm-up", "seconds": dt}


def run_reference(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref, the unmodified
    headers) over every host thread, on the config's signal (c5: a 2^28-sample prefix),
    W warm-up passes, K timed passes, median (bench.hpp:100-122)."""
    world, rank, local = dist_env()
    if rank != 0:
        return
    lib, kind = _ref_lib()
    cfg = args.config
    dtype, n, ks, gen, seed, rows = CONFIGS[cfg]
    threads = os.cpu_count() or 1
    sample = _sample(cfg, args.ref_sample)
    kx = _keyed_input(lib, kind, cfg, sample)
    for _ in range(args.warmup):
        _time_ref(lib, kind, cfg, kx, threads)
    times = []
    outs = 0
    for _ in range(args.steps):
        outs, t = _time_ref(lib, kind, cfg, kx, threads)
        times.append(t)
    med = statistics.median(times)
    value = outs / med
    line = {
        "impl": "reference",
        "metric": "median-filter output samples/sec",
        "value": value,
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": 1e3 * med,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": {"float32": "f32", "float64": "f64", "int32": "i32"}[dtype],
        "data": "synthetic: SplitMix64 recipe of SURVEY.md §8(d), host generated",
        "config": {"workload": WORKLOAD[cfg], "k": list(ks), "sample_samples": sample,
                   "same_as_gpu_config": sample >= n * rows, "timing": "median of K passes"},
        "cpu_baseline": {"value": value, "unit": "samples/s", "cores": threads, "kind": kind,
                         "sample": _sample_text(cfg, sample, threads)},
        "e2e": {"value": value, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the output fold_checksums")
    ap.add_argument("--no-gather", action="store_true", help="skip the (untimed) final gather at N > 1")
    ap.add_argument("--cpu-sample", type=int, default=1 << 26)
    ap.add_argument("--ref-sample", type=int, default=1 << 28)
    ap.add_argument("--n-per-gpu", type=int, default=None,
                    help="override the config's samples per GPU (per row for c3); tests and quick runs only")
    args = ap.parse_args()
    if args.n_per_gpu:
        dtype, n, ks, gen, seed, rows = CONFIGS[args.config]
        CONFIGS[args.config] = (dtype, args.n_per_gpu, ks, gen, seed, rows)
        WORKLOAD[args.config] += f" [n per GPU overridden to {args.n_per_gpu}]"
    if args.warmup < 3 and args.impl == "ours":
        print("note: warmup raised to 3 (timing rules)", file=sys.stderr)
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
