"""Build libbrng.so in-tree with nvcc for sm_100a (no JIT cache, no torch ext).

The shared library travels to the GPU box with the repo snapshot; the
Python binding loads exactly this file.
"""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libbrng.so")
SOURCES = ["brng.cpp", "fill.cu", "gamma.cu", "gibbs.cu", "lda.cu"]
HEADERS = ["brng_internal.h", "philox.cuh"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-fvisibility=hidden",
         "-cudart", "shared", "--expt-relaxed-constexpr"]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    deps.append(os.path.join(ROOT, "include", "brng.h"))
    deps.append(os.path.join(ROOT, "include", "brng_device.cuh"))
    deps.append(os.path.join(ROOT, "include", "brng_device_tables.cuh"))
    deps.append(__file__)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False, out: str | None = None,
          defines: tuple = (), tag: str = "") -> str:
    """Compile libbrng.so (or `out`, with extra -D `defines`, for experiments)."""
    lib = out or LIB
    if out is None and not force and not _stale():
        return LIB
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, src + (f".{tag}" if tag else "") + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, *[f"-D{d}" for d in defines], "-I",
               os.path.join(ROOT, "include"), "-c",
               "-x", "cu", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = lib + ".tmp"
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    import sys
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
