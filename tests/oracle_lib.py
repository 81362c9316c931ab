"""ctypes bindings for the CPU checker (TEST INFRASTRUCTURE ONLY).

Loads ``oracle/libmedfilt_oracle.so`` (the C restatement, oracle/medfilt_oracle.c)
and, when built, ``oracle/_ref/libmedfilt_ref.so`` (the unmodified reference
headers behind oracle/ref_driver.cpp).  Only tests/, ``__graft_entry__.smoke()``
and bench.py's CPU legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORACLE_SO = os.path.join(ORACLE_DIR, "libmedfilt_oracle.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libmedfilt_ref.so")

_u64 = C.c_uint64
_p = C.c_void_p


def build() -> None:
    """Build the checker (and the reference shim when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


class Oracle:
    """The C restatement (oracle/medfilt_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = L = C.CDLL(path)
        for name in ("orc_median_filter_i64", "orc_median_filter_i32", "orc_median_filter_f32",
                     "orc_median_filter_f64", "orc_naive_i64", "orc_piecewise_sort_i64"):
            getattr(L, name).argtypes = [_p, _u64, _u64, _p]
            getattr(L, name).restype = C.c_int
        L.orc_median_filter_trace_i64.argtypes = [_p, _u64, _u64, _p, _p]
        L.orc_median_filter_threads_i64.argtypes = [_p, _u64, _u64, _p, C.c_int]
        L.orc_window_spec.argtypes = [_u64, _u64, _p, _p, _p]
        for name in ("orc_fold_checksum_i64", "orc_fold_checksum_i32"):
            getattr(L, name).argtypes = [_p, _u64]
            getattr(L, name).restype = C.c_uint64
        L.orc_gen_uniform_f64.argtypes = [_u64, _p, _u64]
        L.orc_gen_uniform_f32.argtypes = [_u64, _p, _u64]
        L.orc_gen_mod_i32.argtypes = [_u64, _u64, _p, _u64]
        L.orc_gen_trend_f64.argtypes = [_u64, _p, _u64]
        L.orc_generate_i64.argtypes = [C.c_int, _u64, _u64, C.c_int, _p]
        L.orc_splitmix64.argtypes = [_u64, _p, _u64]

    # -- filters -------------------------------------------------------------------------
    def window_spec(self, n: int, k: int):
        h, b, o = _u64(), _u64(), _u64()
        st = self.lib.orc_window_spec(n, k, C.byref(h), C.byref(b), C.byref(o))
        return st, h.value, b.value, o.value

    def median_filter(self, x: np.ndarray, k: int) -> np.ndarray:
        """Dancing-links restatement; dtype in {int32, int64, float32, float64}."""
        x = np.ascontiguousarray(x)
        st, _, _, keep = self.window_spec(x.size, k)
        if st:
            raise ValueError(f"oracle status {st}")
        y = np.empty(max(keep, 1), dtype=x.dtype)
        fn = {np.dtype(np.int64): self.lib.orc_median_filter_i64,
              np.dtype(np.int32): self.lib.orc_median_filter_i32,
              np.dtype(np.float32): self.lib.orc_median_filter_f32,
              np.dtype(np.float64): self.lib.orc_median_filter_f64}[x.dtype]
        st = fn(_ptr(x), x.size, k, _ptr(y))
        if st:
            raise ValueError(f"oracle status {st}")
        return y[:keep]

    def median_filter_trace(self, x: np.ndarray, k: int):
        x = np.ascontiguousarray(x, dtype=np.int64)
        st, _, _, keep = self.window_spec(x.size, k)
        y = np.empty(max(keep, 1), dtype=np.int64)
        tr = np.zeros((max(keep, 1), 4), dtype=np.uint32)
        st = self.lib.orc_median_filter_trace_i64(_ptr(x), x.size, k, _ptr(y), _ptr(tr))
        assert st == 0
        return y[:keep], tr[:keep]

    def median_filter_threads(self, x: np.ndarray, k: int, threads: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.int64)
        st, _, _, keep = self.window_spec(x.size, k)
        y = np.empty(max(keep, 1), dtype=np.int64)
        st = self.lib.orc_median_filter_threads_i64(_ptr(x), x.size, k, _ptr(y), threads)
        assert st == 0
        return y[:keep]

    def naive(self, x: np.ndarray, k: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.int64)
        st, _, _, keep = self.window_spec(x.size, k)
        y = np.empty(max(keep, 1), dtype=np.int64)
        assert self.lib.orc_naive_i64(_ptr(x), x.size, k, _ptr(y)) == 0
        return y[:keep]

    def piecewise_sort(self, x: np.ndarray, k: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.int64)
        st, _, b, _ = self.window_spec(x.size, k)
        perms = np.empty(b * k, dtype=np.uint32)
        assert self.lib.orc_piecewise_sort_i64(_ptr(x), x.size, k, _ptr(perms)) == 0
        return perms.reshape(b, k)

    # -- checksums / keys ------------------------------------------------------------------
    def fold_checksum(self, v: np.ndarray) -> int:
        v = np.ascontiguousarray(v)
        if v.dtype == np.int32:
            return int(self.lib.orc_fold_checksum_i32(_ptr(v), v.size))
        if v.dtype == np.int64:
            return int(self.lib.orc_fold_checksum_i64(_ptr(v), v.size))
        if v.dtype == np.float32:
            return self.fold_checksum(keymap(v))
        if v.dtype == np.float64:
            return self.fold_checksum(keymap(v))
        raise TypeError(v.dtype)

    # -- generators ------------------------------------------------------------------------
    def uniform_f64(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.lib.orc_gen_uniform_f64(seed, _ptr(out), n)
        return out

    def uniform_f32(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float32)
        self.lib.orc_gen_uniform_f32(seed, _ptr(out), n)
        return out

    def mod_i32(self, seed: int, mod: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.int32)
        self.lib.orc_gen_mod_i32(seed, mod, _ptr(out), n)
        return out

    def trend_f64(self, seed: int, n: int) -> np.ndarray:
        out = np.empty(n, dtype=np.float64)
        self.lib.orc_gen_trend_f64(seed, _ptr(out), n)
        return out

    def generate(self, kind: int, n: int, seed: int, width: int = 64) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        assert self.lib.orc_generate_i64(kind, n, seed, width, _ptr(out)) == 0
        return out if width == 64 else out.astype(np.int32)


def keymap(v: np.ndarray) -> np.ndarray:
    """IEEE bits -> signed totalOrder key.  Integer arrays pass through."""
    if v.dtype == np.float32:
        s = v.view(np.int32)
        return np.where(s >= 0, s, s ^ np.int32(0x7FFFFFFF)).astype(np.int32)
    if v.dtype == np.float64:
        s = v.view(np.int64)
        return np.where(s >= 0, s, s ^ np.int64(0x7FFFFFFFFFFFFFFF)).astype(np.int64)
    return v


def unkey(key: np.ndarray, dtype) -> np.ndarray:
    """Inverse of keymap: signed key -> IEEE value of `dtype` (the map is an involution on bits)."""
    dtype = np.dtype(dtype)
    if dtype == np.float32:
        s = key.astype(np.int32)
        return np.where(s >= 0, s, s ^ np.int32(0x7FFFFFFF)).astype(np.int32).view(np.float32)
    if dtype == np.float64:
        s = key.astype(np.int64)
        return np.where(s >= 0, s, s ^ np.int64(0x7FFFFFFFFFFFFFFF)).astype(np.int64).view(np.float64)
    return key.astype(dtype)


class Reference:
    """The unmodified reference (oracle/_ref/libmedfilt_ref.so)."""

    @staticmethod
    def available() -> bool:
        return os.path.exists(REF_SO)

    def __init__(self, path: str = REF_SO):
        self.lib = L = C.CDLL(path)
        for name in ("ref_median_filter_i32", "ref_median_filter_i64", "ref_naive_i64"):
            getattr(L, name).argtypes = [_p, C.c_size_t, C.c_size_t, _p, _p]
            getattr(L, name).restype = C.c_int
        for name in ("ref_median_filter_threads_i32", "ref_median_filter_threads_i64"):
            getattr(L, name).argtypes = [_p, C.c_size_t, C.c_size_t, _p, C.c_int]
            getattr(L, name).restype = C.c_int
        L.ref_median_filter_rows_i32.argtypes = [_p, C.c_size_t, C.c_size_t, C.c_size_t, _p, C.c_int]
        L.ref_piecewise_sort_i64.argtypes = [_p, C.c_size_t, C.c_size_t, _p]
        L.ref_fold_checksum_i32.argtypes = [_p, C.c_size_t]
        L.ref_fold_checksum_i32.restype = C.c_uint64
        L.ref_fold_checksum_i64.argtypes = [_p, C.c_size_t]
        L.ref_fold_checksum_i64.restype = C.c_uint64
        L.ref_generate_i64.argtypes = [C.c_int, C.c_size_t, C.c_uint64, C.c_int, _p]
        L.ref_last_error.restype = C.c_char_p
        L.ref_run_verify.argtypes = [C.c_size_t, C.c_size_t, C.c_uint64, C.c_int, _p, _p]
        L.ref_sort_via_median_filter_i64.argtypes = [_p, C.c_size_t, C.c_size_t, _p]

    def median_filter(self, x: np.ndarray, k: int) -> np.ndarray:
        """reference median_filter<int32|int64>; floats go through the key map."""
        x = np.ascontiguousarray(x)
        if x.dtype in (np.float32, np.float64):
            return unkey(self.median_filter(keymap(x), k), x.dtype)
        y = np.empty(max(x.size, 1), dtype=x.dtype)
        ylen = C.c_size_t()
        fn = self.lib.ref_median_filter_i32 if x.dtype == np.int32 else self.lib.ref_median_filter_i64
        st = fn(_ptr(x), x.size, k, _ptr(y), C.byref(ylen))
        if st:
            raise ValueError(self.lib.ref_last_error().decode())
        return y[: ylen.value]

    def median_filter_threads(self, x: np.ndarray, k: int, threads: int) -> np.ndarray:
        x = np.ascontiguousarray(x)
        n = x.size
        keep = max(n - k + 1, 0)
        y = np.empty(max(keep, 1), dtype=x.dtype)
        fn = self.lib.ref_median_filter_threads_i32 if x.dtype == np.int32 else self.lib.ref_median_filter_threads_i64
        st = fn(_ptr(x), n, k, _ptr(y), threads)
        if st:
            raise ValueError(self.lib.ref_last_error().decode())
        return y[:keep]

    def median_filter_rows(self, x: np.ndarray, k: int, threads: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.int32)
        rows, ln = x.shape
        keep = max(ln - k + 1, 0)
        y = np.empty((rows, max(keep, 1)), dtype=np.int32)
        assert self.lib.ref_median_filter_rows_i32(_ptr(x), rows, ln, k, _ptr(y), threads) == 0
        return y[:, :keep]

    def piecewise_sort(self, x: np.ndarray, k: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.int64)
        b = -(-x.size // k)
        perms = np.empty(b * k, dtype=np.uint32)
        assert self.lib.ref_piecewise_sort_i64(_ptr(x), x.size, k, _ptr(perms)) == 0
        return perms.reshape(b, k)

    def naive(self, x: np.ndarray, k: int) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.int64)
        y = np.empty(max(x.size, 1), dtype=np.int64)
        ylen = C.c_size_t()
        assert self.lib.ref_naive_i64(_ptr(x), x.size, k, _ptr(y), C.byref(ylen)) == 0
        return y[: ylen.value]

    def fold_checksum(self, v: np.ndarray) -> int:
        v = np.ascontiguousarray(v)
        if v.dtype in (np.float32, np.float64):
            v = keymap(v)
        if v.dtype == np.int32:
            return int(self.lib.ref_fold_checksum_i32(_ptr(v), v.size))
        return int(self.lib.ref_fold_checksum_i64(_ptr(v), v.size))

    def generate(self, kind: int, n: int, seed: int, width: int = 64) -> np.ndarray:
        out = np.empty(n, dtype=np.int64)
        st = self.lib.ref_generate_i64(kind, n, seed, width, _ptr(out))
        if st:
            raise ValueError(self.lib.ref_last_error().decode())
        return out if width == 64 else out.astype(np.int32)

    def run_verify(self, n_max: int, trials: int, seed: int, inject_fault: bool = False):
        e, r = C.c_size_t(), C.c_size_t()
        ok = self.lib.ref_run_verify(n_max, trials, seed, int(inject_fault), C.byref(e), C.byref(r))
        return bool(ok), e.value, r.value

    def sort_via_median_filter(self, blocks: np.ndarray) -> np.ndarray:
        blocks = np.ascontiguousarray(blocks, dtype=np.int64)
        nb, h1 = blocks.shape
        out = np.empty_like(blocks)
        assert self.lib.ref_sort_via_median_filter_i64(_ptr(blocks), nb, h1 - 1, _ptr(out)) == 0
        return out
