"""CPU checks of the C ABI library: it is built for sm_100a, loads, exports every
symbol include/medfilt_gpu.h declares, and its host-side logic (validation, errors,
window arithmetic, kernel-class choice) matches the reference without a GPU."""
from __future__ import annotations

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_1406_1717_b200 as mf
from paper_1406_1717_b200 import _native as N

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "medfilt_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(mf_[a-z0-9_]+)\s*\(", src))


def test_library_exports_header():
    L = N.lib()
    declared = header_symbols()
    assert declared == set(N.EXPORTS), declared ^ set(N.EXPORTS)
    for name in declared:
        assert hasattr(L, name), name


def test_library_is_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_(\d+a?)", out))
    assert arches == {"100a"}, arches


def test_window_spec_and_errors():
    assert mf.make_window_spec(6, 3) == mf.WindowSpec(6, 3, 1, 2)
    assert mf.make_window_spec(5, 3).b == 2
    assert mf.make_window_spec(2, 3).output_size() == 0                  # n < k: empty
    cases = [((0, 3), "input must not be empty"), ((5, 0), "window size must be positive"),
             ((4, 4), "even window size unsupported (window must be k = 2h+1)"),
             ((9, 2**32 - 1), "window size too large")]
    for args, msg in cases:
        with pytest.raises(mf.InvalidArgument) as e:
            mf.make_window_spec(*args)
        assert str(e.value) == msg
    # validation order is the reference's: n == 0 is reported before an even k
    with pytest.raises(mf.InvalidArgument, match="^input must not be empty$"):
        mf.make_window_spec(0, 4)


def test_host_entry_validates_before_device():
    """Argument errors surface identically with no GPU present (no device is touched)."""
    L = N.lib()
    x = np.arange(4, dtype=np.int32)
    y = np.empty(4, dtype=np.int32)
    ylen = C.c_size_t()
    st = L.mf_median_filter(None, N.MF_I32, x.ctypes.data, 4, 3, y.ctypes.data, 4, C.byref(ylen))
    assert st == N.MF_BAD_ARG
    h = C.c_void_p()
    st = L.mf_context_create(0, C.byref(h))
    assert st in (N.MF_OK, N.MF_NO_DEVICE)
    if st == N.MF_NO_DEVICE:
        with pytest.raises(mf.CudaError):
            mf.Context(0)


def test_kernel_classes():
    assert mf.kernel_class(np.float32, 3) == N.MF_CLASS_SMALL
    assert mf.kernel_class(np.float32, 31) == N.MF_CLASS_SMALL
    assert mf.kernel_class(np.int32, 63) == N.MF_CLASS_SMALL      # 64-bit live masks
    assert mf.kernel_class(np.int32, 65) == N.MF_CLASS_MEDIUM
    assert mf.kernel_class(np.float64, 33) == N.MF_CLASS_MEDIUM   # 64-bit keys stop at 31
    assert mf.kernel_class(np.float32, 65) == N.MF_CLASS_MEDIUM
    assert mf.kernel_class(np.int32, 1023) == N.MF_CLASS_MEDIUM
    assert mf.kernel_class(np.float64, 10001) == N.MF_CLASS_LARGE


def test_status_strings():
    for st in range(9):
        assert N.status_string(st).startswith("MF_")
        assert N.error_message(st)


def test_cpp_wrapper_compiles():
    """include/medfilt/gpu.hpp (FilterFn-shaped wrapper) compiles against the C ABI."""
    src = os.path.join(ROOT, "tests", "cpp", "gpu_hpp_check.cpp")
    out = "/tmp/gpu_hpp_check.o"
    r = subprocess.run(["g++", "-std=c++20", "-Wall", "-Wextra", "-fsyntax-only",
                        f"-I{os.path.join(ROOT, 'include')}", src], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
