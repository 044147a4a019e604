"""GPU parity: the sm_100a kernels (through the C ABI) against the pinned CPU
oracle and the reference's golden outputs.  Bit-exact for latency, curve id,
blocks and waves; NaN positions identical."""

import ctypes as C
import hashlib
import json
import math
import os

import numpy as np
import pytest
import torch

import oracle
from conftest import GOLDEN, dataset, golden_grid_arrays, golden_meta, golden_npz, prepared

pytestmark = pytest.mark.gpu

META = golden_meta()
GRIDS = {g["name"]: g for g in META["grids"]}


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("name", list(GRIDS))
def test_grid_verify_outputs_match_golden(gpu, name):
    from paper_2603_00549_b200 import backend
    meta = GRIDS[name]
    prep = prepared(meta)
    lat, cur, blk, wav = backend.predict_grid_device(prep, verify=True)
    lat, cur, blk, wav = (x.cpu().numpy() for x in (lat, cur, blk, wav))
    gold = golden_grid_arrays(meta)
    idx = gold["idx"] if gold["idx"] is not None else slice(None)
    assert np.array_equal(_bits(lat[idx]), _bits(gold["lat"]))
    assert np.array_equal(cur[idx], gold["curve"])
    assert np.array_equal(blk[idx].view(np.uint64), gold["blocks"])
    assert np.array_equal(wav[idx].view(np.uint64), gold["waves"])
    assert hashlib.sha256(lat.tobytes()).hexdigest() == meta["latency_sha256"]
    assert hashlib.sha256(cur.tobytes()).hexdigest() == meta["curve_sha256"]
    # the fast (non-verify) kernel path must give the same bits
    fast = backend.predict_grid(prep)
    assert np.array_equal(_bits(fast), _bits(lat))


@pytest.mark.parametrize("name", ["mk_grid", "matmul_bf16", "exact_mix_bf16", "cutlass_attn_bf16"])
def test_grid_batch_slices_are_independent(gpu, name):
    from paper_2603_00549_b200 import backend
    prep = prepared(GRIDS[name])
    full = backend.predict_grid(prep)
    nb = len(prep.grid.axes["batch"])
    inner = prep.grid.cardinality // nb
    for lo in range(nb):
        for hi in range(lo + 1, nb + 1):
            part = backend.predict_grid_device(prep, b_lo=lo, b_hi=hi).cpu().numpy()
            assert np.array_equal(_bits(part), _bits(full[lo * inner:hi * inner]))


def test_reference_ffi_dropin_slice(gpu):
    """pm2l_predict_grid_slice with the reference's exact argument list (packed
    keys, np.log2 candidate logs as PreparedGrid.tables() builds them) equals
    the reference's compiled Cython kernel (oracle/_ref) or the oracle."""
    from paper_2603_00549_b200 import _native
    lib = _native.load()
    mod = oracle.reference_kernels()
    for name in ("parity_fp32", "matmul_bf16", "exact_mix_fp32", "attn_fp32"):
        prep = prepared(GRIDS[name])
        t = dict(prep.tables())
        recs = prep.records
        # the reference's own candidate logs (nascache.py:189-191)
        t["log_m"] = np.log2(np.array([r.shape.m for r in recs], np.float64))
        t["log_n"] = np.log2(np.array([r.shape.n for r in recs], np.float64))
        t["log_k"] = np.log2(np.array([r.shape.k for r in recs], np.float64))
        B, M, N, K = prep.axis_arrays()
        nb = len(B)
        for lo, hi, pin in ((0, nb, False), (nb - 1, nb, False), (0, nb, True)):
            n_out = (hi - lo) * len(M) * len(N) * len(K)
            # pageable output: staged drain; page-locked: one direct D2H copy
            out = (torch.full((n_out,), -1.0, dtype=torch.float64, pin_memory=True).numpy()
                   if pin else np.empty(n_out, np.float64))
            P = lambda a: a.ctypes.data  # noqa: E731
            rc = lib.pm2l_predict_grid_slice(
                P(B), nb, P(M), len(M), P(N), len(N), P(K), len(K), lo, hi,
                P(t["exact_keys"]), P(t["exact_curve"]), len(recs), P(t["log_m"]), P(t["log_n"]),
                P(t["log_k"]), P(t["cand_curve"]), P(t["sample_offsets"]), P(t["sample_dims"]),
                P(t["sample_thrs"]), len(t["sample_offsets"]) - 1, P(t["ref_dim"]),
                P(t["ref_dur"]), P(t["ref_thr"]), P(t["ref_waves"]), P(t["tile_m"]),
                P(t["tile_n"]), P(t["split_k"]), P(t["blocks_per_wave"]),
                P(t["family_rowblock"]), P(out))
            _native.check(rc, "pm2l_predict_grid_slice")
            want = oracle.grid(t, (B, M, N, K), lo, hi, verify=False)
            assert np.array_equal(_bits(out), _bits(want))
            if mod is not None and lo == 0:
                ref = oracle.reference_predict_grid(mod, t, (B, M, N, K), jobs=2)
                assert np.array_equal(_bits(out), _bits(ref))


def test_unresolved_grid_is_all_nan(gpu):
    from paper_2603_00549_b200 import backend
    prep = prepared(GRIDS["unresolved_bf16_on_fp32"])
    lat, cur, blk, wav = (x.cpu().numpy() for x in backend.predict_grid_device(prep, verify=True))
    assert np.isnan(lat).all() and (cur == -1).all() and (wav == 0).all()
    assert _bits(lat)[0] == 0x7FF8000000000000


def _triple(ti):
    from paper_2603_00549_b200.compute import ConfigResolver, WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    t = META["triples"][ti]
    ds = dataset(t["dataset"])
    res = ConfigResolver(ds.config_map, dataset=ds, wm=WaveModel(ds.device.sm_count))
    return res, (t["family"], DType.parse(t["dtype"]), TransposeMode.parse(t["transpose"]))


def test_points_resolution_and_latency_match_golden(gpu):
    from paper_2603_00549_b200 import _device, _native
    z = golden_npz("points")
    for ti in range(len(META["triples"])):
        sel = np.nonzero(z["triple"] == ti)[0]
        res, triple = _triple(ti)
        shapes = np.stack([z["b"][sel], z["m"][sel], z["n"][sel], z["k"][sel]], 1)
        rec, match, dist = res.resolve_batch(*triple, shapes)
        recs, clist, rec_curve, _, dt = res.triple_tables(*triple)
        curve = np.array([rec_curve[r] for r in rec], np.int32)
        assert np.array_equal(curve, z["curve"][sel])
        assert np.array_equal(match, z["match"][sel])
        # full device predict (latency, waves) through pm2l_points_predict
        dev = _device.device()
        s = _device.to_device(shapes.astype(np.uint32), dev)
        n = len(sel)
        lat = _device.empty(n, "float64", dev)
        cur = _device.empty(n, "int32", dev)
        wav = _device.empty(n, "int32", dev)
        _native.check(_native.load().pm2l_points_predict(
            dt.handle, _native.ptr(s), n, _native.ptr(lat), _native.ptr(cur), _native.ptr(wav),
            0, 0, 0, _device.stream()), "points")
        assert np.array_equal(_bits(lat.cpu().numpy()), _bits(z["lat"][sel]))
        assert np.array_equal(cur.cpu().numpy(), z["curve"][sel])
        assert np.array_equal(wav.cpu().numpy().astype(np.uint64), z["waves"][sel])
        # distances equal the oracle's (ResolvedConfig.distance)
        tables = res.triple_tables(*triple)
        o = oracle.points(__import__("paper_2603_00549_b200.tables", fromlist=["x"])
                          .build_triple_tables(res._records, res._dataset.curves, *triple,
                                               res._wm)[4], shapes)
        assert np.array_equal(_bits(dist), _bits(o[5]))
        assert np.array_equal(rec, o[4])


def test_mode_x_matches_predict_generic_golden(gpu):
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.compute import WaveModel, predict_curve_batch
    z = golden_npz("points")
    ds = dataset("bf16")
    t = next(t for t in META["triples"] if t["dataset"] == "bf16" and t["family"] == "matmul")
    res, triple = _triple(META["triples"].index(t))
    _, clist, _, _, _ = res.triple_tables(*triple)
    shapes = z["modex_shapes"]
    wm = WaveModel(ds.device.sm_count)
    for ci in range(len(clist)):
        lat, _, _ = predict_curve_batch(shapes, clist, np.full(len(shapes), ci), wm)
        assert np.array_equal(_bits(lat), _bits(z["modex_lat"][ci]))


def test_grid_all_curves_matches_oracle(gpu):
    from paper_2603_00549_b200 import backend
    for name in ("matmul_bf16", "cutlass_attn_bf16", "mk_grid"):
        prep = prepared(GRIDS[name])
        allc = backend.predict_grid_all_curves(prep).cpu().numpy()
        B, M, N, K = prep.axis_arrays()
        pts = np.array(list(prep.grid.iter_points()), np.uint32)
        for ci, c in enumerate(prep.curve_list):
            want, _, _ = oracle.points_curve(prep.tables(), pts, np.full(len(pts), ci))
            assert np.array_equal(_bits(allc[ci]), _bits(want))


def test_membound_matches_golden(gpu):
    from paper_2603_00549_b200.membound import MemBoundModel, predict_membound_batch
    from paper_2603_00549_b200.core import DType
    z = golden_npz("membound")
    models = [MemBoundModel(n, DType.FP32, tuple(w), float(b), "d", 0.0, 0.0)
              for n, w, b in zip(("softmax", "gelu", "add"), z["weights"], z["intercept"])]
    for fl in np.unique(z["floor"]):
        sel = z["floor"] == fl
        lat, floored = predict_membound_batch(models, z["features"][sel], z["model"][sel],
                                              [fl] * 3)
        assert np.array_equal(_bits(lat), _bits(z["lat"][sel]))


def test_segment_fsum_equals_math_fsum(gpu):
    from paper_2603_00549_b200.aggregate import segment_fsum
    rng = np.random.default_rng(9)
    lens = rng.integers(0, 70, 3000)
    lens[:5] = [0, 1, 2, 33, 64]
    offs = np.concatenate([[0], np.cumsum(lens)])
    v = rng.uniform(1e-3, 1e4, offs[-1]) * 10.0 ** rng.integers(-6, 9, offs[-1])
    # wide dynamic range (> window) in a few segments -> exact fallback path
    v[offs[7]] = 1e300
    v[offs[9]:offs[10]] = 2.0 ** -1000
    got = segment_fsum(v, offs)
    want = np.array([math.fsum(v[offs[i]:offs[i + 1]]) for i in range(len(lens))])
    assert np.array_equal(_bits(got), _bits(want))
    # exact halfway cases
    v = np.array([1.0, 2.0 ** -53, 2.0 ** -106, 1.0, 2.0 ** -53, 1.0, 2 ** -53, 2 ** -60])
    o = np.array([0, 3, 5, 8])
    want = [math.fsum(v[o[i]:o[i + 1]]) for i in range(3)]
    assert np.array_equal(_bits(segment_fsum(v, o)), _bits(np.array(want)))


def test_predict_model_matches_golden(gpu):
    from paper_2603_00549_b200.aggregate import predict_models
    from paper_2603_00549_b200.ingest import model_graph_from_json_obj
    with open(os.path.join(GOLDEN, "models.json")) as fh:
        gold = json.load(fh)
    ds = dataset(gold["dataset"])
    graphs = [model_graph_from_json_obj(m["graph"]) for m in gold["models"]]
    res = predict_models(graphs, ds)
    for r, m in zip(res, gold["models"]):
        assert r.total_latency_us.hex() == m["total_hex"]
        assert [lp.prediction.latency_us.hex() for lp in r.per_layer] == m["per_layer_hex"]
        assert [lp.predictor_kind for lp in r.per_layer] == m["kinds"]
        assert [list(f) for f in r.flags] == m["flags"]


def test_precompute_store_bytes_match_reference(gpu, tmp_path):
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import CacheStore, GridSpec, precompute
    store = META["store"]
    for name in ("mk_grid", "attn_fp32"):
        meta = GRIDS[name]
        ds = dataset(meta["dataset"])
        grid = GridSpec.from_json_obj(meta["grid"])
        out = tmp_path / f"{name}.bin"
        summary = precompute(grid, ds, WaveModel(ds.device.sm_count), out)
        data = out.read_bytes()
        assert hashlib.sha256(data).hexdigest() == store[name]["sha256"]
        assert summary.backend == "cuda"
        with CacheStore(out) as st:
            st.verify(dataset=ds, grid=grid)
            assert len(st) == grid.cardinality


def test_large_grid_against_reference_and_oracle_sample(gpu):
    """C2-shaped BF16 grid at full size: oracle on a seeded sample of points,
    the compiled reference (oracle/_ref) on a 1M-point sub-grid, plus
    size-independent properties."""
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid
    from paper_2603_00549_b200.core import DType, TransposeMode
    ds = dataset("bf16")
    grid = GridSpec("matmul", DType.BF16, TransposeMode.NN, {
        "batch": (1, 2, 4, 8), "m": tuple(range(64, 64 + 61 * 50, 61)),
        "n": tuple(range(96, 96 + 53 * 50, 53)), "k": tuple(range(32, 32 + 17 * 1000, 17))})
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    lat, cur, blk, wav = backend.predict_grid_device(prep, verify=True)
    lat = lat.cpu().numpy()
    cur = cur.cpu().numpy()
    assert not np.isnan(lat).any() and (lat > 0).all()
    rng = np.random.default_rng(1)
    idx = np.sort(rng.choice(grid.cardinality, 20000, replace=False))
    pts = np.stack(np.unravel_index(idx, grid.shape()), 1)
    shapes = np.stack([np.array(grid.axes[a], np.uint32)[pts[:, i]]
                       for i, a in enumerate(("batch", "m", "n", "k"))], 1)
    o_lat, o_cur, o_wav, *_ = oracle.points(prep.tables(), shapes)
    assert np.array_equal(_bits(lat[idx]), _bits(o_lat))
    assert np.array_equal(cur[idx], o_cur)
    # fast path == verify path, whole grid
    fast = backend.predict_grid(prep)
    assert np.array_equal(_bits(fast), _bits(lat))
    # compiled reference on the first 2 batch values x 25 m values (1.25M points)
    mod = oracle.reference_kernels()
    if mod is not None:
        sub = GridSpec("matmul", DType.BF16, TransposeMode.NN, {
            "batch": (1, 2), "m": grid.axes["m"][:25], "n": grid.axes["n"], "k": grid.axes["k"]})
        sp = PreparedGrid(ds, sub, WaveModel(ds.device.sm_count))
        t = dict(sp.tables())
        ref = oracle.reference_predict_grid(mod, t, sp.axis_arrays(), jobs=os.cpu_count() or 1)
        got = backend.predict_grid(sp)
        assert np.array_equal(_bits(got), _bits(ref))


def test_no_cpu_fallback_flag(gpu):
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.errors import BackendUnavailable
    with pytest.raises(BackendUnavailable):
        backend.predict_grid(prepared(GRIDS["mk_grid"]), force_python=True)


def test_sharded_predict_over_nccl_matches_single_process(gpu, tmp_path):
    """The §8e multi-GPU host path on the device: NCCL process group (one
    rank on the test box), GPU slab prediction, stats all-gather, rank-0
    gather and store write."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2603_00549_b200 import backend, shard
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import write_store
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        meta = GRIDS["exact_mix_bf16"]
        prep = prepared(meta)
        res = shard.predict_sharded(prep, gather=True)
        ref = backend.predict_grid(prep)
        assert np.array_equal(_bits(res.full_numpy()), _bits(ref))
        assert res.full.is_cuda and res.local.is_cuda   # device-resident gather
        assert res.first_unresolved == -1 and res.unresolved == 0
        ds = dataset(meta["dataset"])
        a, b = tmp_path / "a.bin", tmp_path / "b.bin"
        shard.precompute_sharded(prep.grid, ds, WaveModel(ds.device.sm_count), a)
        write_store(b, prep.grid, ds, ref)
        assert a.read_bytes() == b.read_bytes()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", list(GRIDS))
def test_device_store_encoder_matches_host_encoder(gpu, name):
    """pm2l_store_encode == the host encoder (the
    reference's record bytes, nascache.py:325-333), slabs included."""
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.nascache import encode_records, encode_records_device
    prep = prepared(GRIDS[name])
    lat = backend.predict_grid_device(prep)
    host = encode_records(prep.grid, lat.cpu().numpy())
    dev = encode_records_device(prep.grid, lat)
    assert dev.tobytes() == host.tobytes()
    nb = len(prep.grid.axes["batch"])
    if nb > 1:
        inner = prep.grid.cardinality // nb
        part = encode_records_device(prep.grid, lat[inner:], b_lo=1)
        all_host = lat.cpu().numpy()
        from paper_2603_00549_b200.nascache import GridSpec
        sub = GridSpec(prep.grid.family, prep.grid.dtype, prep.grid.transpose_mode,
                       dict(prep.grid.axes, batch=tuple(prep.grid.axes["batch"][1:])))
        assert part.tobytes() == encode_records(sub, all_host[inner:]).tobytes()


def test_device_store_encoder_compacts_unresolved_points(gpu):
    """Random tables with kernels lacking curves: NaN points are dropped and
    the survivors keep canonical order (skip_unresolved)."""
    import torch
    from test_gpu_random_tables import random_tables
    from paper_2603_00549_b200 import _native
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.nascache import GridSpec, encode_records, encode_records_device
    rng = np.random.default_rng(5)
    t, pm, pn, pk = random_tables(rng, 300, 20, 40)
    dt = _native.DeviceTables(t, 0)
    B = np.array([1, 2, 3, 5], np.uint64)
    M = np.array(sorted(set(rng.integers(1, 6000, 9).tolist())), np.uint64)
    N = np.array(sorted(set(rng.integers(1, 6000, 7).tolist())), np.uint64)
    K = np.array(sorted(set(rng.integers(1, 30000, 700).tolist())), np.uint64)
    plan = _native.GridPlan(dt, (B, M, N, K))
    lat = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    plan.launch(lat)
    host_lat = lat.cpu().numpy()
    assert np.isnan(host_lat).any() and not np.isnan(host_lat).all()
    grid = GridSpec("matmul", DType.BF16, TransposeMode.NN,
                    {"batch": tuple(int(x) for x in B), "m": tuple(int(x) for x in M),
                     "n": tuple(int(x) for x in N), "k": tuple(int(x) for x in K)})
    assert encode_records_device(grid, lat).tobytes() == encode_records(grid, host_lat).tobytes()


@pytest.mark.parametrize("sparse", [False, True])
def test_batched_store_lookup_matches_scalar_lookup(gpu, tmp_path, sparse):
    """CacheStore.lookup_many == lookup (nascache.py:408-424)
    point by point: dense stores are direct-indexed, sparse ones searched;
    absent points are NaN or raise MissingEntry naming the first one."""
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.errors import MissingEntry
    from paper_2603_00549_b200.nascache import CacheStore, point_at, write_store
    meta = GRIDS["exact_mix_bf16"]
    prep = prepared(meta)
    lat = backend.predict_grid(prep)
    rng = np.random.default_rng(3)
    if sparse:
        lat = lat.copy()
        lat[rng.choice(len(lat), len(lat) // 3, replace=False)] = np.nan
    path = tmp_path / "s.bin"
    write_store(path, prep.grid, dataset(meta["dataset"]), lat)
    with CacheStore(path) as st:
        pts = np.array([point_at(prep.grid, i) for i in range(prep.grid.cardinality)], np.uint64)
        extra = pts[rng.choice(len(pts), 50)].copy()
        extra[:, 3] += 1  # mostly absent points
        q = np.concatenate([pts, extra])
        got = st.lookup_many(q, missing="nan")
        for i, p in enumerate(q):
            try:
                ref = st.lookup(*(int(v) for v in p))
                assert got[i].view(np.uint64) == np.float64(ref).view(np.uint64)
            except MissingEntry:
                assert np.isnan(got[i])
        want = lat.view(np.uint64)
        present = ~np.isnan(lat)
        assert np.array_equal(got[:len(pts)][present].view(np.uint64), want[present])
        absent = np.nonzero(np.isnan(got))[0]
        if len(absent):
            with pytest.raises(MissingEntry) as exc:
                st.lookup_many(q)
            b, m, n, k = (int(v) for v in q[absent[0]])
            assert f"batch={b} m={m} n={n} k={k}" in str(exc.value)


def test_device_table_set_serves_mixed_grids(gpu):
    """Grids of several triples through one DeviceTableSet: each triple's
    tables are uploaded once and predictions equal fresh PreparedGrids'."""
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid
    from paper_2603_00549_b200.staging import DeviceTableSet
    ds = dataset("bf16")
    st = DeviceTableSet(ds)
    assert st.stage_all() == len(st.triples())
    handles = {}
    for fam, dt, tm in st.triples():
        for ks in ((32, 700, 4096), (100, 9000)):
            grid = GridSpec(fam, dt, tm, {"batch": (1, 3), "m": (64, 200, 1000), "n": (96, 512),
                                          "k": ks})
            prep = st.prepared(grid, ds)
            handles.setdefault((fam, dt, tm), set()).add(id(prep.device_tables(0)))
            got = backend.predict_grid(prep)
            want = backend.predict_grid(PreparedGrid(ds, grid, WaveModel(ds.device.sm_count)))
            assert np.array_equal(_bits(got), _bits(want))
    assert all(len(v) == 1 for v in handles.values())


def test_predict_model_grid_matches_predict_models(gpu):
    """The array-native NAS-grid path (template + shape/feature arrays) gives
    the same per-layer latencies and fsum totals as predict_models."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(GOLDEN), "..", "tools"))
    import c4
    from paper_2603_00549_b200.aggregate import TemplateLayer, predict_model_grid, predict_models
    from paper_2603_00549_b200.core import DType
    ds = dataset("fp32_full")
    params = [(b, s, h, r) for b in (1, 3, 16) for s in (64, 500, 2048) for h in (256, 768, 1280)
              for r in (2, 4)]
    fams = ("linear", "linear", "linear", "batched_matmul", "utility:softmax", "linear", "linear",
            "linear")
    template = [TemplateLayer(i, f, DType.FP32) for i, f in zip(c4.TEMPLATE_IDS, fams)]
    shapes, feats = c4.grid_arrays(params)
    lat, tot = predict_model_grid(template, shapes, feats, ds)
    res = predict_models([c4.block(*p) for p in params], ds)
    for i, r in enumerate(res):
        assert tot[i].hex() == r.total_latency_us.hex()
        assert [x.hex() for x in lat[i]] == [lp.prediction.latency_us.hex() for lp in r.per_layer]
