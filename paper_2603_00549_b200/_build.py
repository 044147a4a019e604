"""Build the sm_100a shared library in-tree (no JIT cache; the .so travels to
the GPU box with the repo snapshot).

    python -m paper_2603_00549_b200._build        # or __graft_entry__.build()
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_NAME = "libpm2l_b200.so"
LIB_PATH = os.path.join(PKG, LIB_NAME)
SOURCES = ["csrc/grid.cu", "csrc/points.cu", "csrc/reduce.cu", "csrc/store.cu", "csrc/tables.cpp",
           "csrc/abi.cpp"]
HEADERS = ["csrc/pm2l_internal.h", "csrc/common.cuh", "../include/pm2l.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    # canonical FP64 order: never contract a*b+c into DFMA (the membound FMA
    # chain uses explicit __fma_rn, which this flag does not affect)
    "-fmad=false",
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
    "-shared", "-cudart", "static",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def source_hash() -> str:
    """sha256 over every source/header compiled into the library; embedded in
    the .so (pm2l_source_hash) so a stale binary is refused at load time."""
    import hashlib
    h = hashlib.sha256()
    for p in SOURCES + HEADERS:
        with open(os.path.join(PKG, p), "rb") as fh:
            h.update(p.encode() + b"\0" + fh.read())
    return h.hexdigest()[:32]


def _stale() -> bool:
    if not os.path.exists(LIB_PATH):
        return True
    lib_t = os.path.getmtime(LIB_PATH)
    return any(os.path.getmtime(os.path.join(PKG, p)) > lib_t for p in SOURCES + HEADERS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB_PATH
    tmp = LIB_PATH + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, f"-DPM2L_SOURCE_HASH=\"{source_hash()}\"", *SOURCES, "-o", tmp]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, cwd=PKG, check=True)
    os.replace(tmp, LIB_PATH)
    return LIB_PATH


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
