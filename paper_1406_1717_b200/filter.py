"""Host-side mirror of the reference's median-filter API, backed by the CUDA library.

Reference interface (/root/reference/proj/include/medfilt/):
  make_window_spec(n, k) -> WindowSpec          core.hpp:51-76
  median_filter<T>(span<const T> x, size_t k)   filter.hpp:149-155   (the hot path)
  piecewise_sort(input) -> permutations         filter.hpp:41-54     (phase API)
Same names, same argument meaning and the same error behaviour: the reference throws
std::invalid_argument with fixed texts (core.hpp:63-69); here ``InvalidArgument``
(a ValueError) carries the identical text.  n < k returns an empty output.

Host arrays (numpy) go through the literal drop-in entry ``mf_median_filter`` (H2D,
kernels, D2H).  CUDA tensors (torch) go through the device entries on torch's current
stream, with no host round trip.  There is no CPU fallback anywhere.
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass

import numpy as np

from . import _native as N

_DTYPES = {np.dtype(np.int32): N.MF_I32, np.dtype(np.int64): N.MF_I64,
           np.dtype(np.float32): N.MF_F32, np.dtype(np.float64): N.MF_F64}


class InvalidArgument(ValueError):
    """std::invalid_argument of the reference (core.hpp:63-69)."""


class CudaError(RuntimeError):
    pass


@dataclass(frozen=True)
class WindowSpec:
    """WindowSpec, core.hpp:51-60."""
    n: int
    k: int
    h: int
    b: int

    def padded_size(self) -> int:
        return self.b * self.k

    def output_size(self) -> int:
        return 0 if self.n < self.k else self.n - self.k + 1

    def empty_output(self) -> bool:
        return self.n < self.k


def _check(st: int) -> None:
    if st == N.MF_OK:
        return
    msg = N.error_message(st)
    if st in (N.MF_EMPTY_INPUT, N.MF_K_ZERO, N.MF_K_EVEN, N.MF_K_TOO_LARGE):
        raise InvalidArgument(msg)
    if st == N.MF_BAD_ARG:
        raise ValueError(msg)
    raise CudaError(f"{N.status_string(st)}: {msg}")


def make_window_spec(n: int, k: int) -> WindowSpec:
    """make_window_spec, core.hpp:62-76 (validation order and texts preserved)."""
    h, b = C.c_size_t(), C.c_size_t()
    _check(N.lib().mf_window_spec(n, k, C.byref(h), C.byref(b), None))
    return WindowSpec(n=n, k=k, h=h.value, b=b.value)


class Context:
    """One mf_context (device, stream, grow-only workspace) per CUDA device, or a
    multi-device context (``Context.multi``) whose host-buffer calls shard over devices."""

    _cache: dict[int, "Context"] = {}
    _cache_lock = threading.Lock()

    def __init__(self, device: int = 0, *, devices=None):
        self._h = C.c_void_p()
        if devices is None:
            self.device = device
            _check(N.lib().mf_context_create(device, C.byref(self._h)))
        else:
            devs = [int(d) for d in devices]
            if not devs:
                raise ValueError("device list must not be empty")
            self.device = devs[0]
            arr = (C.c_int * len(devs))(*devs)
            _check(N.lib().mf_context_create_multi(arr, len(devs), C.byref(self._h)))

    @classmethod
    def multi(cls, devices) -> "Context":
        """A context over several devices (mf_context_create_multi): median_filter and
        median_filter_rows shard the signal (halo'd output ranges) or the rows across them."""
        return cls(devices=devices)

    @property
    def devices(self) -> list[int]:
        n = int(N.lib().mf_context_devices(self._h, None, 0))
        arr = (C.c_int * n)()
        N.lib().mf_context_devices(self._h, arr, n)
        return list(arr)

    @classmethod
    def get(cls, device: int = 0) -> "Context":
        with cls._cache_lock:
            if device not in cls._cache:
                cls._cache[device] = Context(device)
            return cls._cache[device]

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def force_class(self, cls: int) -> None:
        """Pin the kernel class (tests use it to drive every class at small sizes)."""
        _check(N.lib().mf_context_set_option(self._h, N.MF_OPT_FORCE_CLASS, cls))

    def pipeline_chunk(self, samples: int) -> None:
        """Largest chunk of the host-buffer pipeline in samples (0 restores the default)."""
        _check(N.lib().mf_context_set_option(self._h, N.MF_OPT_PIPELINE_CHUNK, samples))

    def last_launches(self) -> int:
        return int(N.lib().mf_context_last_launches(self._h))

    def profile(self, on: bool = True) -> None:
        """Record per-phase CUDA events in the device entries (read with last_phases)."""
        _check(N.lib().mf_context_set_option(self._h, N.MF_OPT_PROFILE, int(bool(on))))

    def last_phases(self) -> list[tuple[str, float]]:
        """(phase name, device ms) of the last device-entry call made with profile() on."""
        cap = 64
        names = (C.c_char_p * cap)()
        ms = (C.c_float * cap)()
        n = int(N.lib().mf_context_last_phases(self._h, names, ms, cap))
        return [(names[i].decode(), float(ms[i])) for i in range(min(n, cap))]

    def __del__(self):
        try:
            if self._h:
                N.lib().mf_context_destroy(self._h)
        except Exception:
            pass


def kernel_class(dtype, k: int) -> int:
    return int(N.lib().mf_kernel_class(_DTYPES[np.dtype(dtype)], k))


# ---------------------------------------------------------------------------------------
# host-buffer API (the drop-in for median_filter<T>)
# ---------------------------------------------------------------------------------------
def median_filter(x, k: int, *, ctx: Context | None = None) -> np.ndarray:
    """median_filter<T>(x, k) (filter.hpp:149-155) for a 1-D host array.

    dtype int32/int64 (the reference's T) or float32/float64 (IEEE totalOrder)."""
    x = np.ascontiguousarray(x)
    if x.ndim != 1:
        raise ValueError("median_filter takes a 1-D signal; use median_filter_rows for batches")
    if x.dtype not in _DTYPES:
        raise TypeError(f"unsupported dtype {x.dtype}")
    ctx = ctx or Context.get(0)
    spec = make_window_spec(x.size, k)
    keep = spec.output_size()
    y = np.empty(max(keep, 1), dtype=x.dtype)
    ylen = C.c_size_t()
    _check(N.lib().mf_median_filter(ctx.handle, _DTYPES[x.dtype], x.ctypes.data, x.size, k,
                                    y.ctypes.data, y.size, C.byref(ylen)))
    return y[: ylen.value]


def median_filter_rows(x, k: int, *, ctx: Context | None = None) -> np.ndarray:
    """Independent signals, one per row of a 2-D host array -> rows x (n-k+1)."""
    x = np.asarray(x)
    if x.ndim != 2 or x.dtype not in _DTYPES:
        raise ValueError("median_filter_rows takes a 2-D int32/int64/float32/float64 array")
    if x.strides[1] != x.itemsize:
        x = np.ascontiguousarray(x)
    rows, n = x.shape
    ctx = ctx or Context.get(0)
    spec = make_window_spec(n, k)
    keep = spec.output_size()
    y = np.empty((rows, max(keep, 1)), dtype=x.dtype)
    _check(N.lib().mf_median_filter_rows(ctx.handle, _DTYPES[x.dtype], x.ctypes.data, rows, n,
                                         x.strides[0] // x.itemsize, k, y.ctypes.data, y.shape[1]))
    return y[:, :keep]


# ---------------------------------------------------------------------------------------
# device API (torch CUDA tensors; torch is only the allocator / stream plumbing)
# ---------------------------------------------------------------------------------------
def _torch():
    import torch
    return torch


def _tdt(t) -> int:
    torch = _torch()
    m = {torch.int32: N.MF_I32, torch.int64: N.MF_I64, torch.float32: N.MF_F32, torch.float64: N.MF_F64}
    if t.dtype not in m:
        raise TypeError(f"unsupported dtype {t.dtype}")
    return m[t.dtype]


def _stream_of(t, stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream(t.device)
    return C.c_void_p(stream.cuda_stream)


def median_filter_device(x, k: int, *, out=None, stream=None, ctx: Context | None = None):
    """median_filter on a 1-D CUDA tensor, stream-ordered on torch's current stream."""
    torch = _torch()
    if not x.is_cuda or x.dim() != 1:
        raise ValueError("median_filter_device takes a 1-D CUDA tensor")
    x = x.contiguous()
    spec = make_window_spec(x.numel(), k)
    keep = spec.output_size()
    if out is None:
        out = torch.empty(max(keep, 1), dtype=x.dtype, device=x.device)
    ctx = ctx or Context.get(x.device.index)
    _check(N.lib().mf_median_filter_device(ctx.handle, _tdt(x), C.c_void_p(x.data_ptr()), x.numel(), k,
                                           C.c_void_p(out.data_ptr()), _stream_of(x, stream)))
    return out[:keep]


def median_filter_rows_device(x, k: int, *, out=None, stream=None, ctx: Context | None = None):
    torch = _torch()
    if not x.is_cuda or x.dim() != 2 or x.stride(1) != 1:
        raise ValueError("median_filter_rows_device takes a row-major 2-D CUDA tensor")
    rows, n = x.shape
    keep = make_window_spec(n, k).output_size()
    if out is None:
        out = torch.empty((rows, max(keep, 1)), dtype=x.dtype, device=x.device)
    ctx = ctx or Context.get(x.device.index)
    _check(N.lib().mf_median_filter_rows_device(ctx.handle, _tdt(x), C.c_void_p(x.data_ptr()), rows, n,
                                                x.stride(0), k, C.c_void_p(out.data_ptr()), out.stride(0),
                                                _stream_of(x, stream)))
    return out[:, :keep]


def block_sort_device(x, k: int, *, stream=None, ctx: Context | None = None):
    """piecewise_sort (filter.hpp:41-54) on the device: (b, k) uint32-valued int64 tensor of
    permutations, perms[j, t] = index of the t-th smallest of block j (stable)."""
    torch = _torch()
    x = x.contiguous()
    spec = make_window_spec(x.numel(), k)
    perm = torch.empty(spec.b * k, dtype=torch.int32, device=x.device)
    ctx = ctx or Context.get(x.device.index)
    _check(N.lib().mf_block_sort_device(ctx.handle, _tdt(x), C.c_void_p(x.data_ptr()), x.numel(), k,
                                        C.c_void_p(perm.data_ptr()), _stream_of(x, stream)))
    return perm.view(spec.b, k)


def generate_device(kind: str, seed: int, n: int, *, offset: int = 0, device: int = 0, mod: int = 16,
                    stream=None, ctx: Context | None = None):
    """SplitMix64 inputs generated on the device (bit-identical to the host stream):
    kind in {"uniform_f32", "uniform_f64", "mod_i32"}; element j is stream value offset + j."""
    torch = _torch()
    kinds = {"uniform_f32": (N.MF_GEN_UNIFORM_F32, torch.float32),
             "uniform_f64": (N.MF_GEN_UNIFORM_F64, torch.float64),
             "mod_i32": (N.MF_GEN_MOD_I32, torch.int32)}
    code, dt = kinds[kind]
    out = torch.empty(n, dtype=dt, device=f"cuda:{device}")
    ctx = ctx or Context.get(device)
    _check(N.lib().mf_generate_device(ctx.handle, code, seed, mod, offset, n, C.c_void_p(out.data_ptr()),
                                      _stream_of(out, stream)))
    return out


def fold_checksum(values, state: int = N.MF_FOLD_INIT) -> int:
    """fold_checksum (io.hpp:17-28) of a host array (floats over their totalOrder keys);
    `state` chains: fold_checksum(b, fold_checksum(a)) == fold_checksum(concat(a, b))."""
    v = np.ascontiguousarray(values)
    if v.dtype not in _DTYPES:
        raise TypeError(f"unsupported dtype {v.dtype}")
    return int(N.lib().mf_fold_checksum(_DTYPES[v.dtype], v.ctypes.data, v.size, state))


def generate_trend_f64(seed: int, n: int) -> np.ndarray:
    """Config-4 signal on the host (libm-dependent; see csrc/mf_host.c)."""
    out = np.empty(n, dtype=np.float64)
    N.lib().mf_generate_trend_f64_host(seed, n, out.ctypes.data)
    return out


# ---------------------------------------------------------------------------------------
# §2 lower-bound gadget: sorting through one median-filter call
# ---------------------------------------------------------------------------------------
def _extremes(dtype):
    dt = np.dtype(dtype)
    if dt.kind == "i":
        info = np.iinfo(dt)
        return dt.type(info.min), dt.type(info.max)
    ui = np.uint32 if dt.itemsize == 4 else np.uint64
    # the two ends of IEEE totalOrder: -NaN and +NaN with all-ones payloads
    lo = np.array([~ui(0)], dtype=ui).view(dt)[0]
    hi = np.array([~ui(0) >> ui(1)], dtype=ui).view(dt)[0]
    return lo, hi


def sort_via_median_filter(blocks, h: int | None = None, *, ctx: Context | None = None) -> np.ndarray:
    """sort_via_median_filter (filter.hpp:177-205) on the GPU: every row of `blocks`
    (nb x (h+1)) is surrounded by h below-everything and h above-everything samples, the
    whole gadget is median-filtered with k = 2h+1 in one call, and each block's sorted image
    is read out of the output.  Executable form of the paper's sorting lower bound (§2)."""
    blocks = np.asarray(blocks)
    if blocks.ndim != 2:
        raise ValueError("blocks must be a 2-D array (nb x (h+1))")
    nb, h1 = blocks.shape
    if h is None:
        h = h1 - 1
    if h1 != h + 1:
        raise InvalidArgument("each block must hold h+1 samples")   # filter.hpp:179-181
    if nb == 0:
        return blocks.copy()
    lo, hi = _extremes(blocks.dtype)
    unit = 3 * h + 1
    gadget = np.empty((nb, unit), dtype=blocks.dtype)
    gadget[:, :h] = lo
    gadget[:, h:2 * h + 1] = blocks
    gadget[:, 2 * h + 1:] = hi
    med = median_filter(gadget.ravel(), 2 * h + 1, ctx=ctx)
    # the reference keeps medians[j*unit .. j*unit + h], filter.hpp:199-203
    med = np.concatenate([med, np.empty(unit * nb - med.size, dtype=med.dtype)])
    return med.reshape(nb, unit)[:, :h + 1].copy()
