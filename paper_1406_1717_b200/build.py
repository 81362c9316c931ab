"""Build the CUDA library in-tree: paper_1406_1717_b200/libmedfilt_b200.so.

nvcc cross-compiles for sm_100a only (no other arch, no PTX fallback); the host
generator (csrc/mf_host.c) is compiled by gcc with -ffp-contract=off.  Objects go to
paper_1406_1717_b200/_build/ and the shared library sits next to this file so it
travels with the repo snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(PKG, "_build")
LIB = os.path.join(PKG, "libmedfilt_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC",
                  "-Xcompiler", "-Wall", f"-I{os.path.join(ROOT, 'include')}"]


def _sources():
    cu = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    c = sorted(glob.glob(os.path.join(CSRC, "*.c")))
    hdr = glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(os.path.join(CSRC, "*.h")) + \
        glob.glob(os.path.join(ROOT, "include", "*.h"))
    return cu, c, hdr


def _stale(target: str, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def build(verbose: bool = False, force: bool = False, extra_flags=(), lib: str = LIB, build_dir: str = BUILD) -> str:
    """Compile every source for sm_100a into `lib`.  `extra_flags`/`lib`/`build_dir` build
    experiment variants (e.g. -D switches) side by side with the shipped library."""
    cu, c, hdr = _sources()
    os.makedirs(build_dir, exist_ok=True)
    jobs = []
    objs = []
    for src in cu:
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdr + [__file__]):
            jobs.append([NVCC, *NVFLAGS, *extra_flags, "-c", src, "-o", obj])
    for src in c:
        obj = os.path.join(build_dir, os.path.basename(src) + ".o")
        objs.append(obj)
        if force or _stale(obj, [src] + hdr + [__file__]):
            jobs.append(["gcc", "-O3", "-fPIC", "-ffp-contract=off", "-Wall", "-c", src, "-o", obj])

    def run(cmd):
        if verbose:
            print(" ".join(cmd), flush=True)
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"build failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
        return r.stderr

    with cf.ThreadPoolExecutor(max_workers=max(1, min(8, os.cpu_count() or 1))) as ex:
        for err in ex.map(run, jobs):
            if verbose and err:
                print(err)
    if force or jobs or _stale(lib, objs):
        run([NVCC, *ARCH, "-shared", "-o", lib, *objs, "-lm", "-lcudart"])
    return lib


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force="-f" in sys.argv))
