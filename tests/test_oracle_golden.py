"""Pin the CPU oracle (oracle/pm2l_oracle.c) and the host table builder to the
reference's own outputs (tests/golden/, generated from /root/reference by
make_golden.py).  CPU only."""

import hashlib
import math
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, dataset, golden_grid_arrays, golden_meta, golden_npz, prepared

META = golden_meta()
GRIDS = {g["name"]: g for g in META["grids"]}


def test_dataset_fingerprints_match_reference():
    # SURVEY App. B fingerprints, recomputed by this package's ingest
    for name, fp in META["fingerprints"].items():
        assert dataset(name).fingerprint() == fp
    assert META["fingerprints"]["fp32"].startswith("2dc7f92a197c1f5b")
    assert META["fingerprints"]["bf16"].startswith("a27731db92b6d914")


@pytest.mark.parametrize("name", [g for g in GRIDS if g != "acceptance_100k"])
def test_oracle_grid_matches_reference(name):
    meta = GRIDS[name]
    prep = prepared(meta)
    assert len(prep.records) == meta["n_records"]
    assert len(prep.curve_list) == meta["n_curves"]
    assert prep.fast_path_ok == meta["fast_path_ok"]
    lat, cur, blk, wav = oracle.grid(prep.tables(), prep.axis_arrays())
    gold = golden_grid_arrays(meta)
    idx = gold["idx"] if gold["idx"] is not None else slice(None)
    assert np.array_equal(lat[idx].view(np.uint64), gold["lat"].view(np.uint64))
    assert np.array_equal(cur[idx], gold["curve"])
    assert np.array_equal(blk[idx], gold["blocks"])
    assert np.array_equal(wav[idx], gold["waves"])
    assert hashlib.sha256(lat.tobytes()).hexdigest() == meta["latency_sha256"]
    assert hashlib.sha256(cur.tobytes()).hexdigest() == meta["curve_sha256"]
    assert hashlib.sha256(wav.tobytes()).hexdigest() == meta["waves_sha256"]


def test_oracle_acceptance_grid_sha():
    meta = GRIDS["acceptance_100k"]
    prep = prepared(meta)
    lat, cur, blk, wav = oracle.grid(prep.tables(), prep.axis_arrays())
    assert hashlib.sha256(lat.tobytes()).hexdigest() == meta["latency_sha256"]
    assert hashlib.sha256(wav.tobytes()).hexdigest() == meta["waves_sha256"]


def test_mk_grid_sha_is_survey_appendix_b():
    assert GRIDS["mk_grid"]["latency_sha256"].startswith("0e44bda98fd7f19d")


def test_unpacked_exact_coords_equal_packed_keys():
    # the two exact-match encodings the ABI accepts must agree
    for name in ("exact_mix_fp32", "exact_mix_bf16", "mk_grid"):
        prep = prepared(GRIDS[name])
        a = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
        b = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False, use_coords=True)
        assert np.array_equal(a.view(np.uint64), b.view(np.uint64))


def test_reference_cython_kernel_matches_oracle():
    mod = oracle.reference_kernels()
    if mod is None:
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    for name in ("parity_fp32", "matmul_bf16", "exact_mix_bf16", "attn_fp32"):
        prep = prepared(GRIDS[name])
        ref = oracle.reference_predict_grid(mod, prep.tables(), prep.axis_arrays(), jobs=3)
        ours = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
        assert np.array_equal(ref.view(np.uint64), ours.view(np.uint64))
        # the all-cores CPU baseline (sub-grid calls of the same kernel) is
        # the same function
        for threads in (1, 5):
            tiles = oracle.reference_predict_grid_tiles(mod, prep.tables(), prep.axis_arrays(), threads)
            assert np.array_equal(tiles.view(np.uint64), ref.view(np.uint64))


def _triple_tables(tmeta):
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.tables import build_triple_tables
    ds = dataset(tmeta["dataset"])
    return build_triple_tables(ds.config_map, ds.curves, tmeta["family"],
                               DType.parse(tmeta["dtype"]), TransposeMode.parse(tmeta["transpose"]),
                               WaveModel(ds.device.sm_count))


def test_oracle_points_match_reference_resolver():
    z = golden_npz("points")
    for ti, tmeta in enumerate(META["triples"]):
        sel = np.nonzero(z["triple"] == ti)[0]
        recs, clist, _, _, tables = _triple_tables(tmeta)
        # curve list order must match the reference's PreparedGrid.curve_list
        assert [None if c is None else [c.kernel.algorithm_id, c.kernel.tile_m, c.kernel.tile_n]
                for c in clist] == tmeta["curves"]
        shapes = np.stack([z["b"][sel], z["m"][sel], z["n"][sel], z["k"][sel]], 1)
        lat, cur, wav, mat, rec, dist = oracle.points(tables, shapes)
        assert np.array_equal(lat.view(np.uint64), z["lat"][sel].view(np.uint64))
        assert np.array_equal(cur, z["curve"][sel])
        assert np.array_equal(wav.astype(np.uint64), z["waves"][sel])
        assert np.array_equal(mat, z["match"][sel])


def test_oracle_mode_x_matches_predict_generic():
    z = golden_npz("points")
    tmeta = next(t for t in META["triples"] if t["dataset"] == "bf16" and
                 t["family"] == "matmul")
    _, clist, _, _, tables = _triple_tables(tmeta)
    shapes = z["modex_shapes"]
    for ci in range(len(clist)):
        lat, _, _ = oracle.points_curve(tables, shapes, np.full(len(shapes), ci))
        assert np.array_equal(lat.view(np.uint64), z["modex_lat"][ci].view(np.uint64))


def test_oracle_membound_matches_np_dot():
    z = golden_npz("membound")
    floors = z["floor"]
    # per-op floors: evaluate one model-floor pair at a time
    for fl in np.unique(floors):
        sel = floors == fl
        out, _ = oracle.membound(z["features"][sel], z["model"][sel], z["weights"],
                                 z["intercept"], np.full(3, fl))
        assert np.array_equal(out.view(np.uint64), z["lat"][sel].view(np.uint64))


def test_oracle_fsum_is_math_fsum():
    rng = np.random.default_rng(5)
    for trial in range(300):
        n = int(rng.integers(0, 60))
        v = rng.uniform(1e-3, 1e5, n) * 10.0 ** rng.integers(-8, 8, n)
        assert oracle.segment_fsum(v, [0, n])[0] == math.fsum(v)
    # halfway cases across partials
    v = np.array([1.0, 2.0 ** -53, 2.0 ** -106])
    assert oracle.segment_fsum(v, [0, 3])[0] == math.fsum(v)
