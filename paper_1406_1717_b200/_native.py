"""ctypes binding of libmedfilt_b200.so (the C ABI in include/medfilt_gpu.h).

The library is built in-tree by ``paper_1406_1717_b200.build``.  There is no CPU
fallback: if the library is missing every entry point raises.
"""
from __future__ import annotations

import ctypes as C
import os
import threading

# MF_B200_LIB points at an experiment build (paper_1406_1717_b200.build.build(lib=...))
LIB_PATH = os.environ.get("MF_B200_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "libmedfilt_b200.so")

MF_OK, MF_EMPTY_INPUT, MF_K_ZERO, MF_K_EVEN, MF_K_TOO_LARGE = 0, 1, 2, 3, 4
MF_BAD_ARG, MF_CUDA_ERROR, MF_OUT_OF_MEMORY, MF_NO_DEVICE = 5, 6, 7, 8
MF_I32, MF_I64, MF_F32, MF_F64 = 0, 1, 2, 3
MF_CLASS_AUTO, MF_CLASS_SMALL, MF_CLASS_MEDIUM, MF_CLASS_LARGE = -1, 0, 1, 2
MF_OPT_FORCE_CLASS = 0
MF_OPT_PIPELINE_CHUNK = 1
MF_OPT_PROFILE = 2
MF_GEN_UNIFORM_F32, MF_GEN_UNIFORM_F64, MF_GEN_MOD_I32 = 0, 1, 2

# Every symbol include/medfilt_gpu.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "mf_status_string", "mf_error_message", "mf_window_spec", "mf_kernel_class",
    "mf_context_create", "mf_context_create_multi", "mf_context_devices", "mf_context_destroy",
    "mf_context_set_option", "mf_context_last_launches", "mf_context_last_phases",
    "mf_median_filter", "mf_median_filter_device", "mf_median_filter_rows",
    "mf_median_filter_rows_device", "mf_block_sort_device", "mf_generate_device",
    "mf_generate_trend_f64_host", "mf_fold_checksum",
)
MF_FOLD_INIT = 1469598103934665603

_lock = threading.Lock()
_lib = None


class NativeLibraryMissing(ImportError):
    pass


def lib() -> C.CDLL:
    """Load (once) and return the CUDA library; raise loudly if it is missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise NativeLibraryMissing(
                f"{LIB_PATH} is missing: run `python -m paper_1406_1717_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        sz, vp, u64 = C.c_size_t, C.c_void_p, C.c_uint64
        L.mf_status_string.restype = C.c_char_p
        L.mf_status_string.argtypes = [C.c_int]
        L.mf_error_message.restype = C.c_char_p
        L.mf_error_message.argtypes = [C.c_int]
        L.mf_window_spec.argtypes = [sz, sz, vp, vp, vp]
        L.mf_kernel_class.argtypes = [C.c_int, sz]
        L.mf_context_create.argtypes = [C.c_int, C.POINTER(vp)]
        L.mf_context_create_multi.argtypes = [C.POINTER(C.c_int), C.c_int, C.POINTER(vp)]
        L.mf_context_devices.argtypes = [vp, C.POINTER(C.c_int), C.c_int]
        L.mf_context_destroy.argtypes = [vp]
        L.mf_context_destroy.restype = None
        L.mf_context_set_option.argtypes = [vp, C.c_int, C.c_long]
        L.mf_context_last_launches.argtypes = [vp]
        L.mf_context_last_launches.restype = u64
        L.mf_context_last_phases.argtypes = [vp, C.POINTER(C.c_char_p), C.POINTER(C.c_float), C.c_int]
        L.mf_context_last_phases.restype = C.c_int
        L.mf_median_filter.argtypes = [vp, C.c_int, vp, sz, sz, vp, sz, C.POINTER(sz)]
        L.mf_median_filter_device.argtypes = [vp, C.c_int, vp, sz, sz, vp, vp]
        L.mf_median_filter_rows.argtypes = [vp, C.c_int, vp, sz, sz, sz, sz, vp, sz]
        L.mf_median_filter_rows_device.argtypes = [vp, C.c_int, vp, sz, sz, sz, sz, vp, sz, vp]
        L.mf_block_sort_device.argtypes = [vp, C.c_int, vp, sz, sz, vp, vp]
        L.mf_generate_device.argtypes = [vp, C.c_int, u64, u64, u64, sz, vp, vp]
        L.mf_generate_trend_f64_host.argtypes = [u64, sz, vp]
        L.mf_generate_trend_f64_host.restype = None
        L.mf_fold_checksum.argtypes = [C.c_int, vp, sz, u64]
        L.mf_fold_checksum.restype = u64
        _lib = L
        return L


def status_string(st: int) -> str:
    return lib().mf_status_string(st).decode()


def error_message(st: int) -> str:
    return lib().mf_error_message(st).decode()
