#!/usr/bin/env python3
"""Generate the golden fixtures under tests/golden/ from the REFERENCE itself.

Test infrastructure only.  This script imports the reference package
(`pm2lat`, /root/reference/pkg/src) — which exists only in the build
container, never on the GPU box — builds its Cython kernel in a scratch copy,
and records what the reference computes:

  datasets/*.json     the "shipped profile tables": `oracle.emit_fixture` of the
                      presets fp32(seed 7), bf16(seed 11), generic(seed 13, FP32
                      and BF16), plus fp32 + membound records (seed 23)
                      (reference pm2lat/oracle.py:191-244, 419-473)
  grids.npz           per-grid outputs of backend.predict_grid (Python path and
                      Cython path, asserted bit-identical), with the per-point
                      curve index / blocks / waves / match kind
                      (pm2lat/backend.py:91-113, compute.py:78-106,163-193)
  grids.json          the GridSpecs + metadata (fingerprints, sha256 of outputs)
  points.npz          explicit (shape -> resolve -> predict_generic) samples and
                      shape x every-kernel ("mode X") samples
  membound.npz        fitted models + predict_membound outputs (membound.py:117-127)
  models.json         predict_model per-layer + fsum totals (aggregate.py:173-196)
  store.json          precompute() store sha256 for byte-identity (nascache.py:280-342)

Re-run:  python tests/golden/make_golden.py   (needs /root/reference, Cython, gcc)
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_PKG = os.environ.get("PM2LAT_REFERENCE_PKG", "/root/reference/pkg")


def _import_reference():
    scratch = tempfile.mkdtemp(prefix="pm2lat_ref_")
    dst = os.path.join(scratch, "pkg")
    shutil.copytree(REF_PKG, dst)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=dst,
                   check=True, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
    sys.path.insert(0, os.path.join(dst, "src"))
    import pm2lat  # noqa: F401
    from pm2lat import backend
    assert backend.active_backend() == "cython", "reference Cython kernel did not build"
    return scratch


def main():
    scratch = _import_reference()
    from pm2lat import backend, oracle
    from pm2lat.aggregate import ModelPredictor, predict_model
    from pm2lat.compute import (MATCH_EXACT, WaveModel, block_count, predict_generic,
                                wave_count)
    from pm2lat.core import (DType, LayerSpec, MatMulShape, ModelGraph, TransposeMode)
    from pm2lat.errors import NoConfigAvailable
    from pm2lat.ingest import (dataset_to_json_obj, model_graph_from_json_obj,
                               model_graph_to_json_obj)
    from pm2lat.membound import predict_membound
    from pm2lat.nascache import GridSpec, PreparedGrid, precompute

    os.makedirs(os.path.join(HERE, "datasets"), exist_ok=True)

    # ------------------------------------------------------------ datasets
    fp32_dev = oracle.fp32_device(seed=7)
    bf16_dev = oracle.bf16_device(seed=11)
    gen_dev = oracle.generic_device(seed=13)
    gen_bf16_dev = oracle.generic_device(seed=13, dtype=DType.BF16)
    datasets = {
        "fp32": oracle.emit_fixture(fp32_dev),
        "bf16": oracle.emit_fixture(bf16_dev),
        "generic": oracle.emit_fixture(gen_dev),
        "generic_bf16": oracle.emit_fixture(gen_bf16_dev),
    }
    datasets["fp32_full"] = oracle.with_membound_fixture(datasets["fp32"], count=32, seed=23)
    fingerprints = {}
    from pm2lat.ingest import load_dataset
    for name, ds in list(datasets.items()):
        obj = dataset_to_json_obj(ds)
        path = os.path.join(HERE, "datasets", f"{name}.json")
        with open(path, "w") as fh:
            json.dump(obj, fh, sort_keys=True, separators=(",", ":"))
            fh.write("\n")
        fingerprints[name] = ds.fingerprint()
        # every golden below is computed from the dataset AS LOADED from the
        # committed file (canonical record order), exactly what a consumer of
        # the shipped tables -- and the B200 build's tests -- see
        datasets[name] = load_dataset(path)
        assert datasets[name].fingerprint() == fingerprints[name]

    # ------------------------------------------------------------ grids
    def rng_axes(seed, nb, nm, nn, nk, lo=1, hi=20000):
        r = np.random.default_rng(seed)
        pick = lambda n: tuple(sorted(set(int(v) for v in r.integers(lo, hi, size=n * 3)))[:n])
        return {"batch": tuple(range(1, nb + 1)), "m": pick(nm), "n": pick(nn), "k": pick(nk)}

    FP32, BF16, NN, TN = DType.FP32, DType.BF16, TransposeMode.NN, TransposeMode.TN
    grid_specs = [
        # tests/test_nascache.py:19-25 mk_grid()
        ("mk_grid", "fp32", GridSpec("matmul", FP32, NN, {
            "batch": (1, 2), "m": (64, 100, 128, 1000), "n": (128, 256),
            "k": (32, 500, 2048, 8192)})),
        # tests/test_nascache.py:155-161 compiled-vs-fallback grid
        ("parity_fp32", "fp32", GridSpec("matmul", FP32, NN, {
            "batch": (1, 3), "m": tuple(range(50, 1500, 97)), "n": (64, 200, 512),
            "k": tuple(range(32, 9000, 331))})),
        # tests/test_nascache.py:171-187 row-block family grid
        ("attn_fp32", "generic", GridSpec("flash_attention", FP32, NN, {
            "batch": (48, 96, 192), "k": tuple(range(64, 8192, 501))})),
        ("cutlass_attn_bf16", "generic_bf16", GridSpec("cutlass_attention", BF16, NN, {
            "batch": (8, 12, 96, 640, 4096), "k": tuple(range(17, 20000, 97))})),
        ("linear_fp32", "fp32", GridSpec("linear", FP32, TN, rng_axes(1, 3, 9, 7, 40))),
        ("bmm_fp32", "fp32", GridSpec("batched_matmul", FP32, NN, rng_axes(2, 4, 6, 6, 30))),
        ("matmul_bf16", "bf16", GridSpec("matmul", BF16, NN, {
            "batch": (1, 2, 4, 8), "m": tuple(range(64, 64 + 61 * 12, 61)),
            "n": tuple(range(96, 96 + 53 * 12, 53)), "k": tuple(range(32, 32 + 170 * 50, 170))})),
        ("linear_bf16", "bf16", GridSpec("linear", BF16, TN, rng_axes(3, 2, 10, 10, 25))),
        ("bmm_bf16", "bf16", GridSpec("batched_matmul", BF16, NN, rng_axes(4, 5, 8, 8, 20))),
        # collection shapes: exact hits mixed with nearest (pm2lat/_kernels.pyx:107-114)
        ("exact_mix_fp32", "fp32", GridSpec("matmul", FP32, NN, {
            "batch": (1, 2, 3), "m": (32, 64, 128, 192, 256, 384, 512, 777),
            "n": (32, 64, 128, 256, 512, 600), "k": tuple(2 ** p for p in range(4, 15)) + (100, 3000)})),
        ("exact_mix_bf16", "bf16", GridSpec("batched_matmul", BF16, NN, {
            "batch": (1, 2, 3, 4, 5), "m": (64, 128, 256, 384, 512, 768),
            "n": (64, 128, 256, 512, 768), "k": tuple(2 ** p for p in range(5, 14)) + (48, 5000)})),
        ("triton_mm_fp32", "generic", GridSpec("triton_mm", FP32, NN, rng_axes(5, 2, 8, 8, 20))),
        # wide coordinates (>= 2^16): the reference takes its Python path
        # (nascache.py:163-168); the B200 build serves them natively.
        ("wide_fp32", "fp32", GridSpec("matmul", FP32, NN, {
            "batch": (1, 2), "m": (64, 70000), "n": (64, 100000), "k": (70_000, 80_000, 123)})),
        ("triton_vec_fp32", "generic", GridSpec("triton_vec", FP32, NN, {
            "batch": (1, 7, 64), "k": (1, 100, 4096, 5000, 65536, 70000, 1 << 20, 3 << 20)})),
        # nothing recorded for this triple -> every point unresolved (NaN)
        ("unresolved_bf16_on_fp32", "fp32", GridSpec("matmul", BF16, NN, {
            "batch": (1, 2), "m": (64, 100), "n": (128,), "k": (32, 500)})),
        # tests/test_acceptance.py:261-267 100k-point NAS grid (sha only)
        ("acceptance_100k", "fp32", GridSpec("matmul", FP32, NN, {
            "batch": tuple(range(1, 5)), "m": tuple(range(64, 64 + 25 * 61, 61)),
            "n": tuple(range(96, 96 + 20 * 53, 53)), "k": tuple(range(32, 32 + 50 * 163, 163))})),
    ]

    grids_meta = []
    arrays = {}
    for gname, dsname, grid in grid_specs:
        ds = datasets[dsname]
        wm = WaveModel(sm_count=ds.device.sm_count)
        prep = PreparedGrid(ds, grid, wm)
        lat_py = backend._predict_grid_python(prep)
        if prep.fast_path_ok:
            lat_cy = backend.predict_grid(prep, jobs=3)
            assert np.array_equal(lat_py.view(np.uint64), lat_cy.view(np.uint64)), gname
        n = grid.cardinality
        curve = np.full(n, -1, np.int32)
        blocks = np.zeros(n, np.uint64)
        waves = np.zeros(n, np.uint64)
        match = np.full(n, -1, np.int8)
        for i, (b, m, nn, k) in enumerate(grid.iter_points()):
            shape = MatMulShape(batch=b, m=m, n=nn, k=k)
            try:
                res = prep.resolver.resolve(grid.family, grid.dtype, grid.transpose_mode, shape)
            except NoConfigAvailable:
                continue
            c = ds.curves.get(res.key)
            if c is None:
                continue
            curve[i] = prep._curve_index[res.key]
            match[i] = 0 if res.match == MATCH_EXACT else 1
            blocks[i] = block_count(grid.family, shape, res.key)
            waves[i] = wave_count(shape, res.key, wm.for_curve(c))
        sha = hashlib.sha256(lat_py.tobytes()).hexdigest()
        meta = {"name": gname, "dataset": dsname, "grid": grid.to_json_obj(),
                "sm_count": wm.sm_count, "cardinality": n, "fast_path_ok": prep.fast_path_ok,
                "n_records": len(prep.records), "n_curves": len(prep.curve_list),
                "latency_sha256": sha,
                "curve_sha256": hashlib.sha256(curve.tobytes()).hexdigest(),
                "waves_sha256": hashlib.sha256(waves.tobytes()).hexdigest(),
                "n_nan": int(np.isnan(lat_py).sum()),
                "n_exact": int((match == 0).sum())}
        if n <= 20000:
            arrays[f"{gname}__lat"] = lat_py
            arrays[f"{gname}__curve"] = curve
            arrays[f"{gname}__blocks"] = blocks
            arrays[f"{gname}__waves"] = waves
            arrays[f"{gname}__match"] = match
            meta["full_arrays"] = True
        else:
            # a seeded sample of points keeps the file small
            idx = np.sort(np.random.default_rng(99).choice(n, 4000, replace=False))
            arrays[f"{gname}__idx"] = idx.astype(np.int64)
            arrays[f"{gname}__lat"] = lat_py[idx]
            arrays[f"{gname}__curve"] = curve[idx]
            arrays[f"{gname}__blocks"] = blocks[idx]
            arrays[f"{gname}__waves"] = waves[idx]
            arrays[f"{gname}__match"] = match[idx]
            meta["full_arrays"] = False
        grids_meta.append(meta)
        print(f"grid {gname}: {n} pts, nan={meta['n_nan']} exact={meta['n_exact']}")
    np.savez_compressed(os.path.join(HERE, "grids.npz"), **arrays)

    # ------------------------------------------------------------ explicit points
    # (shape -> ConfigResolver.resolve -> predict_generic), compute.py:150-193,251-268
    prng = np.random.default_rng(2024)
    pts = {k: [] for k in ("ds", "family", "dtype", "transpose", "b", "m", "n", "k",
                           "curve", "lat", "waves", "blocks", "match")}
    ds_names = ["fp32", "bf16", "generic", "generic_bf16"]
    triples_meta = []
    for di, dsname in enumerate(ds_names):
        ds = datasets[dsname]
        wm = WaveModel(sm_count=ds.device.sm_count)
        triples = sorted({(r.family, r.dtype.value, r.transpose_mode.value) for r in ds.config_map})
        for fam, dt, tr in triples:
            grid = GridSpec(fam, DType.parse(dt), TransposeMode.parse(tr), {"k": (1,)})
            prep = PreparedGrid(ds, grid, wm)
            triples_meta.append({"dataset": dsname, "family": fam, "dtype": dt, "transpose": tr,
                                 "curves": [None if c is None else
                                            [c.kernel.algorithm_id, c.kernel.tile_m, c.kernel.tile_n]
                                            for c in prep.curve_list]})
            rowblock = fam in ("triton_vec", "flash_attention", "cutlass_attention")
            shapes = []
            for rec in prep.records[::3]:
                s = rec.shape
                shapes.append((s.batch, s.m, s.n, s.k))
            for _ in range(300):
                if rowblock:
                    shapes.append((int(prng.integers(1, 5000)), 1, 1, int(prng.integers(1, 1 << 21))))
                else:
                    shapes.append((int(prng.integers(1, 17)), int(prng.integers(1, 9000)),
                                   int(prng.integers(1, 9000)), int(prng.integers(1, 20000))))
            for b, m, n, k in shapes:
                shape = MatMulShape(batch=b, m=m, n=n, k=k)
                res = prep.resolver.resolve(fam, DType.parse(dt), TransposeMode.parse(tr), shape)
                c = ds.curves[res.key]
                pred = predict_generic(shape, res.key, c, wm)
                for key, val in (("ds", di), ("family", len(triples_meta) - 1), ("dtype", 0),
                                 ("transpose", 0), ("b", b), ("m", m), ("n", n), ("k", k),
                                 ("curve", prep._curve_index[res.key]), ("lat", pred.latency_us),
                                 ("waves", pred.components["waves"]),
                                 ("blocks", block_count(fam, shape, res.key)),
                                 ("match", 0 if res.match == MATCH_EXACT else 1)):
                    pts[key].append(val)
    points = {
        "triple": np.array(pts["family"], np.int32),
        "b": np.array(pts["b"], np.uint64), "m": np.array(pts["m"], np.uint64),
        "n": np.array(pts["n"], np.uint64), "k": np.array(pts["k"], np.uint64),
        "curve": np.array(pts["curve"], np.int32), "lat": np.array(pts["lat"], np.float64),
        "waves": np.array(pts["waves"], np.uint64), "blocks": np.array(pts["blocks"], np.uint64),
        "match": np.array(pts["match"], np.int8),
    }
    # mode X: every shape x every recorded kernel of the BF16 matmul triple
    ds = datasets["bf16"]
    wm = WaveModel(sm_count=ds.device.sm_count)
    prep = PreparedGrid(ds, GridSpec("matmul", BF16, NN, {"k": (1,)}), wm)
    xs = [(int(prng.integers(1, 9)), int(prng.integers(1, 4000)), int(prng.integers(1, 4000)),
           int(prng.integers(1, 17000))) for _ in range(150)]
    modex = np.zeros((len(prep.curve_list), len(xs)), np.float64)
    for ci, c in enumerate(prep.curve_list):
        for si, (b, m, n, k) in enumerate(xs):
            modex[ci, si] = predict_generic(MatMulShape(b, m, n, k), c.kernel, c, wm).latency_us
    points["modex_shapes"] = np.array(xs, np.uint64)
    points["modex_lat"] = modex
    np.savez_compressed(os.path.join(HERE, "points.npz"), **points)

    # ------------------------------------------------------------ membound
    full = datasets["fp32_full"]
    mp = ModelPredictor(full)
    names = ["softmax", "gelu", "add"]
    models = [mp.membound_model(nm, DType.FP32) for nm in names]
    feats, mids, outs, floors = [], [], [], []
    frng = np.random.default_rng(77)
    for i in range(3000):
        f = oracle.synth_features(frng, log10_lo=0.0 if i % 7 == 0 else 5.0)
        mi = i % 3
        fl = 2.0 if i % 11 else 0.0
        feats.append(f.as_vector())
        mids.append(mi)
        floors.append(fl)
        outs.append(predict_membound(models[mi], f, floor_us=fl).latency_us)
    from pm2lat.core import MemBoundFeatures
    for mi in range(3):   # zero features -> intercept (or floor)
        feats.append((0.0,) * 5)
        mids.append(mi)
        floors.append(2.0)
        outs.append(predict_membound(models[mi], MemBoundFeatures(0, 0, 0, 0, 0)).latency_us)
    np.savez_compressed(
        os.path.join(HERE, "membound.npz"),
        weights=np.array([m.weights for m in models], np.float64),
        intercept=np.array([m.intercept for m in models], np.float64),
        max_rel_err=np.array([m.max_rel_err for m in models], np.float64),
        mean_rel_err=np.array([m.mean_rel_err for m in models], np.float64),
        features=np.array(feats, np.float64), model=np.array(mids, np.int32),
        floor=np.array(floors, np.float64), lat=np.array(outs, np.float64))

    # ------------------------------------------------------------ whole models
    sys.path.insert(0, os.path.join(scratch, "pkg", "tests"))
    from test_ingest import TRANSFORMER_BLOCK
    graphs = [TRANSFORMER_BLOCK]
    grng = np.random.default_rng(33)
    for gi in range(300):
        layers = []
        for li in range(int(grng.integers(1, 9))):
            if grng.random() < 0.2:
                f = oracle.synth_features(grng)
                layers.append(LayerSpec(f"u{li}", "utility:" + names[int(grng.integers(0, 3))],
                                        FP32, features=f))
            else:
                plan = fp32_dev.plans[int(grng.integers(0, 13))]
                shape = plan.collection_shape(int(grng.integers(32, 8192)))
                shape = MatMulShape(batch=shape.batch * int(grng.integers(1, 4)),
                                    m=shape.m, n=shape.n, k=shape.k)
                layers.append(LayerSpec(f"c{li}", plan.key.family, FP32, shape=shape,
                                        transpose_mode=plan.key.transpose_mode))
        graphs.append(model_graph_to_json_obj(ModelGraph(f"g{gi}", tuple(layers))))
    model_out = []
    for gobj in graphs:
        g = model_graph_from_json_obj(gobj)
        res = predict_model(g, full)
        model_out.append({
            "graph": gobj,
            "total_hex": res.total_latency_us.hex(),
            "per_layer_hex": [lp.prediction.latency_us.hex() for lp in res.per_layer],
            "kinds": [lp.predictor_kind for lp in res.per_layer],
            "flags": [list(f) for f in res.flags],
        })
    with open(os.path.join(HERE, "models.json"), "w") as fh:
        json.dump({"dataset": "fp32_full", "models": model_out}, fh, separators=(",", ":"))
        fh.write("\n")

    # ------------------------------------------------------------ store bytes
    store = {}
    for gname in ("mk_grid", "attn_fp32"):
        gname_, dsname, grid = next(g for g in grid_specs if g[0] == gname)
        ds = datasets[dsname]
        path = os.path.join(scratch, f"{gname}.bin")
        precompute(grid, ds, WaveModel(ds.device.sm_count), path)
        with open(path, "rb") as fh:
            data = fh.read()
        store[gname] = {"sha256": hashlib.sha256(data).hexdigest(), "size": len(data)}
    gname_, dsname, grid = next(g for g in grid_specs if g[0] == "unresolved_bf16_on_fp32")
    path = os.path.join(scratch, "partial.bin")
    precompute(grid, datasets[dsname], None, path, skip_unresolved=True)
    with open(path, "rb") as fh:
        data = fh.read()
    store["unresolved_skip"] = {"sha256": hashlib.sha256(data).hexdigest(), "size": len(data)}

    with open(os.path.join(HERE, "grids.json"), "w") as fh:
        json.dump({"fingerprints": fingerprints, "grids": grids_meta, "triples": triples_meta,
                   "store": store}, fh, indent=1, sort_keys=True)
        fh.write("\n")
    shutil.rmtree(scratch, ignore_errors=True)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
