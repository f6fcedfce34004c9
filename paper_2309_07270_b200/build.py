"""Build libxdrop.so in-tree with nvcc for sm_100a (no JIT cache, no torch extension)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libxdrop.so")
# tests only: the same sources with -DXDROP_CHECKED (every packed-pool read bounds-checked, traps)
OUT_CHECKED = os.path.join(HERE, "libxdrop_checked.so")
SOURCES = [os.path.join(CSRC, f) for f in ("xdrop_capi.cu", "xdrop_peaks.cu", "xdrop_filters.cu", "sched.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, f) for f in ("xdrop_kernels.cuh", "xdrop_pk16.cuh", "xdrop_pkwide.cuh", "sched.h")] + [
    os.path.join(os.path.dirname(HERE), "include", "xdrop.h")]
NVCC_FLAGS = ["-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
              "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-shared"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def _build_one(out: str, extra: list, force: bool, verbose: bool) -> str:
    if not force and os.path.exists(out):
        t = os.path.getmtime(out)
        if all(os.path.getmtime(d) <= t for d in DEPS):
            return out
    tmp = out + f".tmp{os.getpid()}"
    cmd = [nvcc(), *NVCC_FLAGS, *extra, *SOURCES, "-o", tmp]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    os.replace(tmp, out)
    return out


def build(force: bool = False, verbose: bool = False) -> str:
    return _build_one(OUT, [], force, verbose)


def build_checked(force: bool = False, verbose: bool = False) -> str:
    return _build_one(OUT_CHECKED, ["-DXDROP_CHECKED"], force, verbose)


def build_all(force: bool = False, verbose: bool = False) -> tuple:
    """libxdrop.so and libxdrop_checked.so, the two nvcc runs concurrently (each is one big
    translation unit, so this halves the wall time of a clean build)."""
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=2) as ex:
        a = ex.submit(build, force, verbose)
        c = ex.submit(build_checked, force, verbose)
        return a.result(), c.result()


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv, verbose=True))
