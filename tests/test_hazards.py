"""Reference numeric hazards pinned by tests/golden/make_golden_hazards.py
(reference-generated):

* log2 source: at 13 integers below 2^16 np.log2 differs
  from libm log2 by one ULP.  The reference's Python path (math.log2 for
  candidates and queries, compute.py:239,261) and its Cython path (np.log2
  candidate tables, nascache.py:189-191) then disagree on exact distance
  ties.  This package's own tables follow the Python path; the reference
  FFI drop-in uses whatever logs its caller passes, so with the reference's
  np.log2 tables it reproduces the Cython path.
* wide coordinates: explicit / per-op resolution of coordinates >= 2^22
  (up to 2^32 - 1; the 16-byte descriptor holds u32) with libm log2 as the
  reference's resolver takes it (compute.py:256-268).
"""

import json
import math
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, dataset

with open(os.path.join(GOLDEN, "hazards.json")) as fh:
    META = json.load(fh)
Z = dict(np.load(os.path.join(GOLDEN, "hazards.npz")))
HAZARDS = META["hazards"]


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _prep():
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid
    ds = dataset("hazard_fp32")
    return PreparedGrid(ds, GridSpec.from_json_obj(META["grid"]), WaveModel(META["sm_count"]))


def _np_log2_tables(prep):
    t = dict(prep.tables())
    for ax in ("m", "n", "k"):
        t[f"log_{ax}"] = np.log2(np.array([getattr(r.shape, ax) for r in prep.records], np.float64))
    return t


def _triple(di):
    from paper_2603_00549_b200.compute import ConfigResolver, WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    ds = dataset(META["datasets"][di])
    res = ConfigResolver(ds.config_map, dataset=ds, wm=WaveModel(ds.device.sm_count))
    return ds, res, (META["families"][di], DType.FP32, TransposeMode.NN)


def _points(di, narrow=True):
    sel = Z["pt_ds"] == di
    shp = np.stack([Z["pt_b"][sel], Z["pt_m"][sel], Z["pt_n"][sel], Z["pt_k"][sel]], 1)
    keep = shp.max(1) < (1 << 32) if narrow else shp.max(1) >= (1 << 32)
    idx = np.nonzero(sel)[0][keep]
    return shp[keep], idx


# ---------------------------------------------------------------- CPU
def test_hazard_integers_are_the_np_log2_libm_disagreements():
    for h in HAZARDS:
        assert float(np.log2(np.float64(h))) != math.log2(h)
    assert META["n_python_ne_cython"] > 0


def test_fingerprint_of_hazard_dataset():
    assert dataset("hazard_fp32").fingerprint() == META["fingerprint"]


def test_oracle_follows_both_reference_paths():
    prep = _prep()
    assert np.array_equal(_bits(oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)),
                          _bits(Z["grid_py"]))
    assert np.array_equal(_bits(oracle.grid(_np_log2_tables(prep), prep.axis_arrays(),
                                            verify=False)), _bits(Z["grid_cy"]))
    assert not np.array_equal(_bits(Z["grid_py"]), _bits(Z["grid_cy"]))


@pytest.mark.parametrize("di", [0, 1, 2])
def test_oracle_wide_coordinate_resolution(di):
    from paper_2603_00549_b200.tables import build_triple_tables
    ds, res, triple = _triple(di)
    shapes, idx = _points(di)
    t = build_triple_tables(ds.config_map, ds.curves, *triple, res._wm)[4]
    lat, cur, wav, mat, rec, dist = oracle.points(t, shapes.astype(np.uint32))
    assert np.array_equal(_bits(lat), _bits(Z["pt_lat"][idx]))
    assert np.array_equal(cur, Z["pt_curve"][idx])
    assert np.array_equal(mat, Z["pt_match"][idx])
    assert np.array_equal(_bits(dist), _bits(Z["pt_dist"][idx]))
    w = Z["pt_waves"][idx]
    assert np.array_equal(wav, np.minimum(w, 0xFFFFFFFF).astype(np.uint32))


# ---------------------------------------------------------------- GPU
@pytest.mark.gpu
def test_grid_paths_follow_their_reference_twins(gpu):
    """Package tables (math.log2) == the reference Python path; the FFI drop-in
    given the reference's own np.log2 tables == the reference Cython path."""
    from conftest import ffi_slice
    from paper_2603_00549_b200 import backend
    prep = _prep()
    assert np.array_equal(_bits(backend.predict_grid(prep)), _bits(Z["grid_py"]))
    B, M, N, K = prep.axis_arrays()
    got = ffi_slice(_np_log2_tables(prep), (B, M, N, K), 0, len(B),
                    np.empty(prep.grid.cardinality, np.float64))
    assert np.array_equal(_bits(got), _bits(Z["grid_cy"]))


@pytest.mark.gpu
@pytest.mark.parametrize("di", [0, 1, 2])
def test_wide_coordinates_resolve_and_predict_like_the_reference(gpu, di):
    """ConfigResolver.resolve_batch + predict_curve_batch (the per-op API that
    predict_model uses) on coordinates up to 2^32 - 1: curve, match,
    distance, latency and waves equal the reference's scalar path."""
    from paper_2603_00549_b200.compute import predict_curve_batch
    ds, res, triple = _triple(di)
    shapes, idx = _points(di)
    rec, match, dist = res.resolve_batch(*triple, shapes)
    recs, clist, rec_curve, _, _ = res.triple_tables(*triple)
    cur = np.array([rec_curve[r] for r in rec], np.int32)
    assert np.array_equal(cur, Z["pt_curve"][idx])
    assert np.array_equal(match, Z["pt_match"][idx])
    assert np.array_equal(_bits(dist), _bits(Z["pt_dist"][idx]))
    lat, waves, _ = predict_curve_batch(shapes, clist, cur, res._wm)
    assert np.array_equal(_bits(lat), _bits(Z["pt_lat"][idx]))
    assert np.array_equal(waves, Z["pt_waves"][idx])


@pytest.mark.gpu
def test_scalar_predict_on_wide_layer(gpu):
    """predict_generic / ConfigResolver.resolve on single wide shapes."""
    from paper_2603_00549_b200.compute import WaveModel, predict_generic
    from paper_2603_00549_b200.core import MatMulShape
    ds, res, triple = _triple(1)
    shapes, idx = _points(1)
    for s, i in list(zip(shapes, idx))[:40]:
        shape = MatMulShape(*(int(x) for x in s))
        r = res.resolve(*triple, shape)
        p = predict_generic(shape, r.key, ds.curves[r.key], WaveModel(ds.device.sm_count))
        assert p.latency_us.hex() == float(Z["pt_lat"][i]).hex()
        assert p.components["waves"] == int(Z["pt_waves"][i])


@pytest.mark.gpu
def test_coordinates_past_u32_are_refused(gpu):
    from paper_2603_00549_b200.errors import ValidationError
    ds, res, triple = _triple(1)
    shapes, _ = _points(1, narrow=False)
    assert len(shapes)
    with pytest.raises(ValidationError):
        res.resolve_batch(*triple, [tuple(int(x) for x in shapes[0])])


@pytest.mark.gpu
def test_points_kernel_hazard_ties(gpu):
    """The tie queries through the explicit-descriptor kernel directly."""
    from paper_2603_00549_b200 import _device, _native
    from paper_2603_00549_b200.tables import build_triple_tables
    ds, res, triple = _triple(0)
    shapes, idx = _points(0)
    recs, clist, rec_curve, _, dt = res.triple_tables(*triple)
    s = _device.to_device(shapes.astype(np.uint32), _device.device())
    n = len(shapes)
    lat = _device.empty(n, "float64", _device.device())
    _native.check(_native.load().pm2l_points_predict(
        dt.handle, _native.ptr(s), n, _native.ptr(lat), 0, 0, 0, 0, 0, _device.stream()),
        "points")
    small = shapes.max(1) < (1 << 22)
    got = _device.to_numpy(lat)
    assert np.array_equal(_bits(got[small]), _bits(Z["pt_lat"][idx][small]))
    assert np.isnan(got[~small]).all()   # no log2 extension given: invalid, not guessed
