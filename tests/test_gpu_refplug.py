"""The reference's OWN code path with the B200 library plugged in.

The unmodified reference package is installed under baseline/_ref
(``pip install --no-index --no-deps --target baseline/_ref <copy of
/root/reference/pkg>``; its compiled Cython
kernel comes with it).  ``paper_2603_00549_b200.refplug.install`` swaps the
INTEGRATION.md binding in as ``pm2lat.backend._kernels`` (backend.py:28-34),
and the reference's own ``precompute`` (nascache.py:280-342) and
``predict_grid`` (backend.py:49-88, batch-slab thread pool included) then
run on the B200 -- compared with the same calls on the reference's Cython
kernel and with the reference-generated golden store hashes."""

import hashlib
import importlib
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT, golden_meta

pytestmark = pytest.mark.gpu
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def pm2lat():
    if not os.path.isdir(os.path.join(REF, "pm2lat")):
        pytest.skip("reference not installed under baseline/_ref")
    if REF not in sys.path:
        sys.path.insert(0, REF)
    mod = importlib.import_module("pm2lat")
    importlib.import_module("pm2lat.backend")
    assert mod.__file__.startswith(REF)
    return mod


@pytest.fixture()
def plugged(pm2lat):
    from paper_2603_00549_b200 import refplug
    prev = refplug.install(pm2lat.backend)
    yield pm2lat
    pm2lat.backend._kernels = prev


def _ds(pm2lat, name):
    return pm2lat.ingest.load_dataset(os.path.join(GOLDEN, "datasets", f"{name}.json"))


def test_reference_precompute_with_b200_plugin_writes_the_golden_store(gpu, plugged, tmp_path):
    pm2lat = plugged
    from pm2lat.nascache import GridSpec, precompute
    meta = golden_meta()
    grids = {g["name"]: g for g in meta["grids"]}
    for name in ("mk_grid", "attn_fp32"):
        g = grids[name]
        ds = _ds(pm2lat, g["dataset"])
        grid = GridSpec.from_json_obj(g["grid"])
        out = tmp_path / f"{name}.bin"
        summary = precompute(grid, ds, None, out, jobs=2)
        assert hashlib.sha256(out.read_bytes()).hexdigest() == meta["store"][name]["sha256"]
        assert summary.total_points == grid.cardinality == summary.entries_written


def test_reference_predict_grid_c2_plugin_equals_its_cython_kernel(gpu, pm2lat):
    """C2 (10 M points) through the reference's own backend.predict_grid with
    its batch-slab thread pool (jobs=4): B200 plugin == Cython kernel."""
    from pm2lat.compute import WaveModel
    from pm2lat.core import DType, TransposeMode
    from pm2lat.nascache import GridSpec, PreparedGrid
    from paper_2603_00549_b200 import refplug
    ds = _ds(pm2lat, "bf16")
    grid = GridSpec("matmul", DType.BF16, TransposeMode.NN, {
        "batch": (1, 2, 4, 8), "m": tuple(range(64, 64 + 61 * 50, 61)),
        "n": tuple(range(96, 96 + 53 * 50, 53)), "k": tuple(range(32, 32 + 17 * 1000, 17))})
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    assert pm2lat.backend._kernels is not None, "reference Cython kernel missing"
    want = pm2lat.backend.predict_grid(prep, jobs=4)
    prev = refplug.install(pm2lat.backend)
    try:
        got = pm2lat.backend.predict_grid(prep, jobs=4)
        got1 = pm2lat.backend.predict_grid(prep, jobs=1)
    finally:
        pm2lat.backend._kernels = prev
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert np.array_equal(got1.view(np.uint64), want.view(np.uint64))
