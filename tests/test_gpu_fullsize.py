"""Parity at the benchmarked configurations, at full size.

Every grid here is the one bench.py / tools/bench_modes.py / tools/c5.py
time, launched whole on the B200 and compared bit for bit against the
reference's own compiled kernel (oracle/_ref: the unmodified
_kernels.pyx:76-133, given the reference's np.log2 candidate tables as
nascache.py:189-191 builds them) over every host core — or, where the
reference kernel would take minutes, on a seeded >= 1 M-point sub-grid of
the full launch (sub-grids are exact: a point's result depends only on its
own coordinates, _kernels.pyx:97-133).  The C oracle covers what the
reference has no batch kernel for (explicit descriptors, mode X)."""

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

import oracle
from conftest import dataset

pytestmark = pytest.mark.gpu

THREADS = max(1, len(os.sched_getaffinity(0)))
B8 = (1, 2, 4, 8, 16, 32, 64, 128)


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _ref_tables(prep):
    """PreparedGrid.tables() with the reference's np.log2 candidate logs."""
    t = dict(prep.tables())
    recs = prep.records
    for ax in ("m", "n", "k"):
        t[f"log_{ax}"] = np.log2(np.array([getattr(r.shape, ax) for r in recs], np.float64))
    return t


def _reference(prep, axes=None):
    """Reference Cython kernel (all host cores) or, if it was not built, the
    C oracle threaded the same way."""
    axes = prep.axis_arrays() if axes is None else axes
    t = _ref_tables(prep)
    mod = oracle.reference_kernels()
    if mod is not None:
        return oracle.reference_predict_grid_tiles(mod, t, axes, THREADS)
    B, M, N, K = (np.ascontiguousarray(a, np.uint64) for a in axes)
    inner = len(M) * len(N) * len(K)
    out = np.empty(len(B) * inner, np.float64)
    cuts = np.linspace(0, len(M), min(len(M), THREADS) + 1, dtype=int)

    def run(b, m0, m1):
        o = oracle.grid(t, (B, M[m0:m1], N, K), b, b + 1, verify=False)
        out[b * inner + m0 * len(N) * len(K):b * inner + m1 * len(N) * len(K)] = o

    with ThreadPoolExecutor(THREADS) as pool:
        list(pool.map(lambda a: run(*a), [(b, int(m0), int(m1)) for b in range(len(B))
                                          for m0, m1 in zip(cuts[:-1], cuts[1:]) if m1 > m0]))
    return out


def _prep(ds_name, family, dtype, tmode, axes):
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid
    ds = dataset(ds_name)
    grid = GridSpec(family, DType.parse(dtype), TransposeMode.parse(tmode), axes)
    return PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))


def _c2_axes():
    return {"batch": (1, 2, 4, 8), "m": tuple(range(64, 64 + 61 * 50, 61)),
            "n": tuple(range(96, 96 + 53 * 50, 53)), "k": tuple(range(32, 32 + 17 * 1000, 17))}


def _sub_index(shape, picks):
    """Flat indices (canonical order) of the sub-grid picks[a] ⊂ axis a."""
    grids = np.meshgrid(*[np.asarray(p, np.int64) for p in picks], indexing="ij")
    return np.ravel_multi_index([g.ravel() for g in grids], shape)


def test_c2_full_grid_equals_reference_kernel(gpu):
    """bench.py's workload, all 10 M points: the device planner path (what
    the bench times), the host-planned path and the reference FFI drop-in
    all equal the reference's compiled kernel."""
    import torch
    from paper_2603_00549_b200 import _native, backend
    from conftest import ffi_slice
    prep = _prep("bf16", "matmul", "bf16", "nn", _c2_axes())
    ref = _reference(prep)
    got = backend.predict_grid(prep)
    if not np.array_equal(_bits(got), _bits(ref)):   # diagnostics for an intermittent mismatch
        dev = backend.predict_grid_device(prep).cpu().numpy()
        again = backend.predict_grid(prep)
        d = np.nonzero(_bits(got) != _bits(ref))[0]
        try:
            from cuda.bindings import runtime as cr
            err, a = cr.cudaPointerGetAttributes(got.ctypes.data)
            kind = (int(err), int(a.type), hex(int(a.hostPointer or 0)), hex(got.ctypes.data))
        except Exception as exc:  # diagnostics only
            kind = repr(exc)
        raise AssertionError(f"pointer attributes of the result {kind}; "
            f"predict_grid mismatch: {len(d)} points, nonzero {np.count_nonzero(got)}, first {d[:4]}, "
            f"device path ok {np.array_equal(_bits(dev), _bits(ref))}, second call ok "
            f"{np.array_equal(_bits(again), _bits(ref))}, 8 MB chunks {sorted(set((d * 8) >> 23))[:12]}")
    # bench.py's plan-inclusive path: device-resident axes, planner kernel
    axes = [torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).cuda()
            for a in prep.axis_arrays()]
    dp = _native.DeviceGridPlanner(prep.device_tables(0), *(len(a) for a in axes))
    out = torch.full((prep.grid.cardinality,), -1.0, dtype=torch.float64, device="cuda")
    dp.launch(axes, out)
    assert dp.kernel_path() == 3, "C2 must take the lookup kernel"
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(ref))
    # the reference's own FFI signature with its own (np.log2) tables
    t = _ref_tables(prep)
    B, M, N, K = prep.axis_arrays()
    ffi = ffi_slice(t, (B, M, N, K), 0, len(B), np.empty(prep.grid.cardinality, np.float64))
    assert np.array_equal(_bits(ffi), _bits(ref))


@pytest.mark.parametrize("family", ["cutlass_attention", "flash_attention"])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_c3_attention_full_grid_equals_reference_kernel(gpu, family, dtype):
    """C3: 28 B*H batch values x seq 64..65535 (1.83 M points per family),
    row-block wave model, lookup ring kernel."""
    bh = sorted({b * h for b in B8 for h in (8, 12, 16, 20, 32, 40, 64)})
    assert len(bh) == 28
    prep = _prep("generic_bf16" if dtype == "bf16" else "generic", family, dtype, "nn",
                 {"batch": tuple(bh), "m": (1,), "n": (1,), "k": tuple(range(64, 65536))})
    from paper_2603_00549_b200 import backend
    got = backend.predict_grid(prep)
    ref = _reference(prep)
    if not np.array_equal(_bits(got), _bits(ref)):   # diagnostics for an intermittent mismatch
        from cuda.bindings import runtime as cr
        err, a = cr.cudaPointerGetAttributes(got.ctypes.data)
        again = backend.predict_grid(prep)
        raise AssertionError(f"C3 predict_grid mismatch: nonzero {np.count_nonzero(got)}, pointer "
                             f"type {int(a.type)}, second call ok "
                             f"{np.array_equal(_bits(again), _bits(ref))}")
    lat, cur, blk, wav = (x.cpu().numpy() for x in backend.predict_grid_device(prep, verify=True))
    assert np.array_equal(_bits(lat), _bits(got))


C5_GEMM = [
    ("matmul", "nn", 100, 100, 8, 7500),
    ("linear", "tn", 50, 100, 12, 5000),
    ("batched_matmul", "nn", 50, 50, 12, 5000),
]


@pytest.mark.parametrize("family,tmode,nm,nn,kstep,nk", C5_GEMM)
def test_c5_gemm_component_shard0(gpu, family, tmode, nm, nn, kstep, nk):
    """C5 GEMM components at tools/c5.py's size: rank 0's shard (batch
    value 1 of 8) launched whole (k chunked by the kernel), checked on a
    seeded 12 x 12 x all-k sub-grid (>= 0.72 M points) against the
    reference kernel, plus every point of the shard finite and > 0."""
    from paper_2603_00549_b200 import backend
    axes = {"batch": B8, "m": tuple(range(64, 64 + 61 * nm, 61)),
            "n": tuple(range(96, 96 + 53 * nn, 53)), "k": tuple(range(32, 32 + kstep * nk, kstep))}
    prep = _prep("bf16", family, "bf16", tmode, axes)
    lat = backend.predict_grid_device(prep, b_lo=0, b_hi=1)
    rng = np.random.default_rng(hash(family) % 2**32)
    mi = np.sort(rng.choice(nm, 12, replace=False))
    ni = np.sort(rng.choice(nn, 12, replace=False))
    idx = _sub_index((1, nm, nn, nk), [[0], mi, ni, np.arange(nk)])
    import torch
    got = lat[torch.from_numpy(idx).cuda()].cpu().numpy()
    B, M, N, K = prep.axis_arrays()
    want = _reference(prep, (B[:1], M[mi], N[ni], K))
    assert np.array_equal(_bits(got), _bits(want))
    assert bool(torch.isfinite(lat).all()) and bool((lat > 0).all())


@pytest.mark.parametrize("family", ["flash_attention", "cutlass_attention"])
def test_c5_attention_component_shard0(gpu, family):
    """C5 attention components: batch' 8..4800 step 8 x seq 64..62563 —
    rank 0's 75-value slab (4.69 M points) compared whole."""
    from paper_2603_00549_b200 import backend
    axes = {"batch": tuple(range(8, 8 + 8 * 600, 8)), "m": (1,), "n": (1,),
            "k": tuple(range(64, 64 + 62500))}
    prep = _prep("generic_bf16", family, "bf16", "nn", axes)
    got = backend.predict_grid_device(prep, b_lo=0, b_hi=75).cpu().numpy()
    B, M, N, K = prep.axis_arrays()
    assert np.array_equal(_bits(got), _bits(_reference(prep, (B[:75], M, N, K))))


def _c2_shapes(n, seed):
    axes = _c2_axes()
    rng = np.random.default_rng(seed)
    pick = [rng.integers(0, len(axes[a]), n) for a in ("batch", "m", "n", "k")]
    return np.stack([np.asarray(axes[a], np.uint32)[p]
                     for a, p in zip(("batch", "m", "n", "k"), pick)], 1)


def _oracle_points_threaded(t, shapes):
    parts = np.array_split(np.arange(len(shapes)), THREADS)
    with ThreadPoolExecutor(THREADS) as pool:
        res = list(pool.map(lambda p: oracle.points(t, shapes[p]), parts))
    return [np.concatenate([r[i] for r in res]) for i in range(6)]


def test_points_mode_c2_shapes_match_oracle(gpu):
    """tools/bench_modes.py 'points': explicit 16-byte descriptors over the
    C2 shapes (2 M seeded ops, exact + nearest + tile/wave + interpolation)
    against the oracle's ConfigResolver restatement: latency, curve, waves,
    match kind, record and distance."""
    import torch
    from paper_2603_00549_b200 import _native
    prep = _prep("bf16", "matmul", "bf16", "nn", _c2_axes())
    shapes = _c2_shapes(2_000_000, 5)
    # mix in every recorded shape so exact hits are exercised
    rec = np.array([r.shape.as_tuple() for r in prep.records], np.uint32)
    shapes[:len(rec)] = rec
    n = len(shapes)
    s = torch.from_numpy(shapes).cuda()
    lat = torch.empty(n, dtype=torch.float64, device="cuda")
    cur = torch.empty(n, dtype=torch.int32, device="cuda")
    wav = torch.empty(n, dtype=torch.int32, device="cuda")
    mat = torch.empty(n, dtype=torch.int8, device="cuda")
    rid = torch.empty(n, dtype=torch.int32, device="cuda")
    dist = torch.empty(n, dtype=torch.float64, device="cuda")
    dt = prep.device_tables(0)
    _native.check(_native.load().pm2l_points_predict(
        dt.handle, s.data_ptr(), n, lat.data_ptr(), cur.data_ptr(), wav.data_ptr(),
        mat.data_ptr(), rid.data_ptr(), dist.data_ptr(), _native.stream_handle()), "points")
    o_lat, o_cur, o_wav, o_mat, o_rec, o_dist = _oracle_points_threaded(prep.tables(), shapes)
    assert np.array_equal(_bits(lat.cpu().numpy()), _bits(o_lat))
    assert np.array_equal(cur.cpu().numpy(), o_cur)
    assert np.array_equal(wav.cpu().numpy().view(np.uint32), o_wav)
    assert np.array_equal(mat.cpu().numpy(), o_mat)
    assert np.array_equal(rid.cpu().numpy(), o_rec)
    assert np.array_equal(_bits(dist.cpu().numpy()), _bits(o_dist))
    assert (o_mat[:len(rec)] == 0).all()


def test_mode_x_full_c2_grid_sample_matches_oracle(gpu):
    """Mode X on the full C2 grid: 10 M shapes x 60 kernels = 600 M pairs on
    the device, 1 M seeded pairs checked against the oracle's predict_generic
    restatement (compute.py:150-193)."""
    import torch
    from paper_2603_00549_b200 import backend
    prep = _prep("bf16", "matmul", "bf16", "nn", _c2_axes())
    allc = backend.predict_grid_all_curves(prep)
    C, P = allc.shape
    assert C == len(prep.curve_list) == 60 and P == 10_000_000
    rng = np.random.default_rng(3)
    ci = rng.integers(0, C, 1_000_000)
    pi = rng.integers(0, P, 1_000_000)
    got = allc[torch.from_numpy(ci).cuda(), torch.from_numpy(pi).cuda()].cpu().numpy()
    axes = _c2_axes()
    coords = np.unravel_index(pi, prep.grid.shape())
    shapes = np.stack([np.asarray(axes[a], np.uint32)[c]
                       for a, c in zip(("batch", "m", "n", "k"), coords)], 1)
    t = prep.tables()
    parts = np.array_split(np.arange(len(ci)), THREADS)
    with ThreadPoolExecutor(THREADS) as pool:
        res = list(pool.map(lambda p: oracle.points_curve(t, shapes[p], ci[p])[0], parts))
    assert np.array_equal(_bits(got), _bits(np.concatenate(res)))
    assert bool(torch.isfinite(allc).all())


def test_c4_nas_grid_matches_reference_predict_model(gpu):
    """C4 (BASELINE configs[3], tools/c4.py): all 2,142 transformer-block
    models through the array path (predict_model_grid: one resolution +
    prediction launch per kernel triple, one membound batch, exact segmented
    fsum) and a seeded subset through the object API (predict_models),
    against the reference's own predict_model (tests/golden/c4.npz,
    make_golden_c4.py): every per-layer latency and every fsum total
    bit-identical."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                    "tools"))
    import c4
    from conftest import GOLDEN
    from paper_2603_00549_b200.aggregate import TemplateLayer, predict_model_grid, predict_models
    from paper_2603_00549_b200.core import DType
    z = np.load(os.path.join(GOLDEN, "c4.npz"))
    params = [tuple(int(x) for x in p) for p in z["params"]]
    ds = dataset("fp32_full")
    fams = ("linear", "linear", "linear", "batched_matmul", "utility:softmax", "linear", "linear",
            "linear")
    template = [TemplateLayer(i, f, DType.FP32) for i, f in zip(c4.TEMPLATE_IDS, fams)]
    shapes, feats = c4.grid_arrays(params)
    lat, totals = predict_model_grid(template, shapes, feats, ds)
    assert np.array_equal(_bits(lat), _bits(z["lat"]))
    assert np.array_equal(_bits(totals), _bits(z["total"]))
    sel = np.random.default_rng(4).choice(len(params), 120, replace=False)
    res = predict_models([c4.block(*params[i]) for i in sel], ds)
    for r, i in zip(res, sel):
        assert r.total_latency_us.hex() == float(z["total"][i]).hex()
        assert [lp.prediction.latency_us.hex() for lp in r.per_layer] == \
            [float(x).hex() for x in z["lat"][i]]


@pytest.mark.parametrize("ds_name,family,dtype,tmode", [
    ("fp32", "matmul", "fp32", "nn"),        # 13-curve FP32 preset
    ("fp32", "linear", "fp32", "tn"),
    ("generic", "triton_mm", "fp32", "nn"),  # the generic preset's triton family
])
def test_c2_shaped_grid_other_tables_full(gpu, ds_name, family, dtype, tmode):
    """The C2 grid shape (10 M points) against the other shipped presets:
    whatever kernel path their tables take (lookup, single or general
    sweep), device-planned and host-planned launches equal the reference's
    compiled kernel point for point."""
    import torch
    from paper_2603_00549_b200 import _native, backend
    prep = _prep(ds_name, family, dtype, tmode, _c2_axes())
    ref = _reference(prep)
    got = backend.predict_grid_device(prep).cpu().numpy()
    assert np.array_equal(_bits(got), _bits(ref))
    axes = [torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).cuda()
            for a in prep.axis_arrays()]
    dp = _native.DeviceGridPlanner(prep.device_tables(0), *(len(a) for a in axes))
    out = torch.empty(prep.grid.cardinality, dtype=torch.float64, device="cuda")
    dp.launch(axes, out)
    torch.cuda.synchronize()
    assert dp.status() == 0
    assert np.array_equal(_bits(out.cpu().numpy()), _bits(ref))
    dp.close()


@pytest.mark.parametrize("ds_name,family,dtype,tmode", [
    ("fp32", "matmul", "fp32", "nn"),
    ("fp32", "batched_matmul", "fp32", "nn"),
    ("generic", "triton_mm", "fp32", "nn"),
    ("generic_bf16", "flash_attention", "bf16", "nn"),
])
def test_points_mode_other_presets_match_oracle(gpu, ds_name, family, dtype, tmode):
    """Explicit descriptors against the other shipped presets (their tables
    take the row walk, the member pass or the general k-group sweep): 1 M
    seeded ops with every recorded shape mixed in, all outputs vs the
    oracle's ConfigResolver restatement."""
    import torch
    from paper_2603_00549_b200 import _native
    prep = _prep(ds_name, family, dtype, tmode, _c2_axes())
    rng = np.random.default_rng(11)
    n = 1_000_000
    shapes = np.stack([rng.integers(1, 300, n), rng.integers(1, 9000, n),
                       rng.integers(1, 9000, n), rng.integers(1, 70000, n)], 1).astype(np.uint32)
    rec = np.array([r.shape.as_tuple() for r in prep.records], np.uint32)
    shapes[:len(rec)] = rec
    s = torch.from_numpy(shapes).cuda()
    outs = [torch.empty(n, dtype=x, device="cuda") for x in
            (torch.float64, torch.int32, torch.int32, torch.int8, torch.int32, torch.float64)]
    _native.check(_native.load().pm2l_points_predict(
        prep.device_tables(0).handle, s.data_ptr(), n, *[o.data_ptr() for o in outs],
        _native.stream_handle()), "points")
    o_lat, o_cur, o_wav, o_mat, o_rec, o_dist = _oracle_points_threaded(prep.tables(), shapes)
    lat, cur, wav, mat, rid, dist = (o.cpu().numpy() for o in outs)
    assert np.array_equal(_bits(lat), _bits(o_lat))
    assert np.array_equal(cur, o_cur)
    assert np.array_equal(wav.view(np.uint32), o_wav)
    assert np.array_equal(mat, o_mat)
    assert np.array_equal(rid, o_rec)
    assert np.array_equal(_bits(dist), _bits(o_dist))


def test_membound_c5_sized_batch_matches_oracle(gpu):
    """tools/bench_modes.py 'membound' / C5's membound share: 5 M feature
    vectors over 32 fitted-shape models (wide dynamic range, floors hit and
    missed, negative weights) -- the left-to-right FMA chain and the floor
    bit for bit against the oracle."""
    from paper_2603_00549_b200.core import DType
    from paper_2603_00549_b200.membound import MemBoundModel, predict_membound_batch
    rng = np.random.default_rng(23)
    n, nm = 5_000_000, 32
    f = np.exp(rng.uniform(0, 40, (n, 5)))
    ids = rng.integers(0, nm, n).astype(np.int32)
    w = rng.uniform(-1e-9, 4e-9, (nm, 5))
    b = rng.uniform(-5, 5, nm)
    floors = rng.uniform(0.5, 3.0, nm)
    models = [MemBoundModel(f"k{i}", DType.FP32, tuple(w[i]), float(b[i]), "d", 0.0, 0.0)
              for i in range(nm)]
    lat, flo = predict_membound_batch(models, f, ids, floors)
    o_lat, o_flo = oracle.membound(f, ids, w, b, floors)
    assert np.array_equal(_bits(lat), _bits(o_lat))
    assert np.array_equal(flo, o_flo)
    assert 0 < flo.mean() < 1   # both sides of the floor are exercised


def test_segment_fsum_many_models_matches_math_fsum(gpu):
    """Per-model totals at NAS-grid scale: 200 k segments of 0..40 terms
    (empty, single-term, signed, wide dynamic range, exact cancellations)
    equal math.fsum bit for bit (the reference's aggregate.py:193)."""
    from paper_2603_00549_b200.aggregate import segment_fsum
    rng = np.random.default_rng(29)
    nseg = 200_000
    lens = rng.integers(0, 41, nseg)
    off = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    n = int(off[-1])
    v = rng.standard_normal(n) * np.exp(rng.uniform(-30, 30, n))
    # exact cancellations in every 97th segment
    for s in range(0, nseg, 97):
        a, b = off[s], off[s + 1]
        if b - a >= 2:
            v[b - 1] = -v[a]
    got = segment_fsum(v, off)
    want = oracle.segment_fsum(v, off)
    assert np.array_equal(_bits(got), _bits(want))


def test_c2_store_records_device_equal_host_encoder(gpu):
    """§8f row 1 at C2 size: the 10 M store records (400 MB, big-endian
    coordinates + latency) encoded on the device equal the host encoder's
    bytes (digest compared)."""
    import hashlib
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.nascache import encode_records, encode_records_device
    prep = _prep("bf16", "matmul", "bf16", "nn", _c2_axes())
    lat = backend.predict_grid_device(prep)
    dev = encode_records_device(prep.grid, lat)
    host = encode_records(prep.grid, lat.cpu().numpy())
    assert dev.nbytes == host.nbytes == 40 * prep.grid.cardinality
    assert hashlib.sha256(dev.tobytes()).digest() == hashlib.sha256(host.tobytes()).digest()


def test_c2_store_batched_lookup_returns_the_written_latencies(gpu, tmp_path):
    """§8f row 2 at C2 size: the 10 M-record store written from the device
    result; 1 M batched lookups (random points, the first and last record)
    return exactly the latencies at those points, and an absent point raises
    MissingEntry as CacheStore.lookup does."""
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.errors import MissingEntry
    from paper_2603_00549_b200.nascache import CacheStore, encode_records_device, write_store
    prep = _prep("bf16", "matmul", "bf16", "nn", _c2_axes())
    lat_d = backend.predict_grid_device(prep)
    path = str(tmp_path / "c2.store")
    write_store(path, prep.grid, prep.dataset, records=encode_records_device(prep.grid, lat_d))
    lat = lat_d.cpu().numpy()
    shape = prep.grid.shape()
    rng = np.random.default_rng(41)
    idx = np.concatenate([[0, len(lat) - 1], rng.integers(0, len(lat), 1_000_000)])
    coords = np.stack(np.unravel_index(idx, shape), 1)
    axes = [np.asarray(prep.grid.axes[a], np.uint64) for a in ("batch", "m", "n", "k")]
    pts = np.stack([axes[i][coords[:, i]] for i in range(4)], 1)
    with CacheStore(path) as st:
        got = st.lookup_many(pts)
        assert np.array_equal(_bits(got), _bits(lat[idx]))
        with pytest.raises(MissingEntry):
            st.lookup_many(np.array([[3, 64, 96, 32]], np.uint64))   # batch 3 is not on the grid
