#!/bin/bash
# Build the library of git revision $1 into paper_2603_00549_b200/libpm2l_$2.so
# (A/B timing on one GPU box: PM2L_LIB_PATH=... python bench.py)
set -e
cd "$(dirname "$0")/.."
REV=$1; TAG=$2
TMP=$(mktemp -d)
git archive "$REV" paper_2603_00549_b200 include | tar -x -C "$TMP"
python - "$TMP" "$TAG" <<'PY'
import os, subprocess, sys
tmp, tag = sys.argv[1], sys.argv[2]
out = os.path.join(os.getcwd(), "paper_2603_00549_b200", f"libpm2l_{tag}.so")
sys.path.insert(0, tmp)  # the revision's own build script and source list
from paper_2603_00549_b200 import _build
if "out_path" in _build.build.__code__.co_varnames:
    _build.build(force=True, out_path=out)
else:
    subprocess.run([_build.nvcc(), *_build.NVCC_FLAGS, *_build.SOURCES, "-o", out], cwd=_build.PKG, check=True)
print(out)
PY
rm -rf "$TMP"
