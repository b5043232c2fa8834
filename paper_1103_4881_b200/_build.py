"""Build libds.so in-tree with nvcc for sm_100a (no JIT cache: the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB = os.path.join(PKG, "libds.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-std=c++17", "-O3", "-lineinfo",
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-Xcompiler", "-fPIC,-fvisibility=hidden",
    "-shared",
]


def sources():
    return sorted(glob.glob(os.path.join(PKG, "csrc", "*.cu")) +
                  glob.glob(os.path.join(PKG, "csrc", "*.cuh")) +
                  glob.glob(os.path.join(PKG, "csrc", "*.h")) +
                  [os.path.join(ROOT, "include", "ds.h")])


def stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(s) > t for s in sources())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile every csrc/*.cu to an object in parallel, then link libds.so."""
    if not force and not stale():
        return LIB
    from concurrent.futures import ThreadPoolExecutor

    cu = [s for s in sources() if s.endswith(".cu")]
    tag = f".tmp{os.getpid()}"
    flags = [f for f in NVCC_FLAGS if f != "-shared"]
    if verbose:
        flags = ["-Xptxas=-v", *flags]

    def compile_one(src):
        obj = os.path.join(PKG, "csrc", os.path.basename(src) + tag + ".o")
        subprocess.check_call([NVCC, *flags, "-I", os.path.join(ROOT, "include"), "-c", src, "-o", obj])
        return obj

    with ThreadPoolExecutor(max_workers=len(cu)) as ex:
        objs = list(ex.map(compile_one, cu))
    tmp = LIB + tag
    try:
        subprocess.check_call([NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared",
                               "-Xcompiler", "-fPIC", *objs, "-o", tmp])
        os.replace(tmp, LIB)
    finally:
        for o in objs:
            if os.path.exists(o):
                os.remove(o)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
