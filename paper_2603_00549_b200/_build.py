"""Build the sm_100a shared library in-tree (no JIT cache; the .so travels to
the GPU box with the repo snapshot).

    python -m paper_2603_00549_b200._build        # or __graft_entry__.build()

Every source is compiled to its own object in parallel (the lookup kernel is
split into one translation unit per batch-slab width for this), objects are
cached under build/obj by a hash of (source, headers, flags), then linked.
"""

from __future__ import annotations

import hashlib
import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
LIB_NAME = "libpm2l_b200.so"
LIB_PATH = os.path.join(PKG, LIB_NAME)
OBJ_DIR = os.path.join(ROOT, "build", "obj")
SOURCES = ["csrc/grid.cu", "csrc/grid_sweep.cu", "csrc/grid_single.cu", "csrc/grid_lookup_nb1.cu",
           "csrc/grid_lookup_nb2.cu", "csrc/grid_lookup_nb4.cu", "csrc/grid_lookup_nb8.cu",
           "csrc/plan.cu", "csrc/points.cu", "csrc/audit.cu", "csrc/reduce.cu", "csrc/store.cu",
           "csrc/tables.cpp", "csrc/abi.cpp"]
HEADERS = ["csrc/pm2l_internal.h", "csrc/common.cuh", "csrc/grid_common.cuh",
           "csrc/grid_lookup.cuh", "../include/pm2l.h"]

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = [
    *ARCH, "-O3", "-lineinfo", "-std=c++17",
    # canonical FP64 order: never contract a*b+c into DFMA (the membound FMA
    # chain uses explicit __fma_rn, which this flag does not affect)
    "-fmad=false",
    "-Xcompiler", "-fPIC,-O2,-ffp-contract=off",
]
LINK_FLAGS = [*ARCH, "-shared", "-cudart", "static",]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found")


def source_hash() -> str:
    """sha256 over every source/header compiled into the library; embedded in
    the .so (pm2l_source_hash) so a stale binary is refused at load time."""
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


def _compile(src: str, flags: list[str], verbose: bool) -> str:
    h = hashlib.sha256(" ".join(flags).encode())
    for p in [src] + HEADERS:
        with open(os.path.join(PKG, p), "rb") as fh:
            h.update(fh.read())
    obj = os.path.join(OBJ_DIR, os.path.basename(src) + "." + h.hexdigest()[:16] + ".o")
    if os.path.exists(obj):
        return obj
    tmp = obj + f".{os.getpid()}.tmp"
    cmd = [nvcc(), *flags, "-c", src, "-o", tmp]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, cwd=PKG, check=True)
    os.replace(tmp, obj)
    return obj


def build(force: bool = False, verbose: bool = False, extra_flags: list[str] | None = None,
          out_path: str | None = None) -> str:
    """Compile (in parallel, cached per object) and link the library.
    extra_flags / out_path: diagnostic builds (e.g. -DPM2L_TIMING) into
    another file."""
    out_path = out_path or LIB_PATH
    if not force and not extra_flags and out_path == LIB_PATH and not _stale():
        return LIB_PATH
    os.makedirs(OBJ_DIR, exist_ok=True)
    flags = [*NVCC_FLAGS, f"-DPM2L_SOURCE_HASH=\"{source_hash()}\"", *(extra_flags or [])]
    # abi.cpp alone embeds the source hash; the other objects stay cached
    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(
            s, flags if s.endswith("abi.cpp") else [f for f in flags if "PM2L_SOURCE_HASH" not in f],
            verbose), SOURCES))
    tmp = out_path + ".tmp"
    subprocess.run([nvcc(), *LINK_FLAGS, *objs, "-o", tmp], cwd=PKG, check=True)
    os.replace(tmp, out_path)
    return out_path


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
