"""Randomised tables (not from a dataset): many k-groups (> 32 exercises the
general nearest path), coordinate lattices that force distance ties, records
whose kernel has no curve (NaN), row-block and GEMM curves — GPU grid and
explicit-descriptor kernels against the C oracle, bit for bit."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def random_tables(rng, R, C, n_k_values, rowblock=False, wide=False, lattice=False):
    pool_m = rng.choice(np.arange(1, 5000), size=12, replace=False)
    pool_n = rng.choice(np.arange(1, 5000), size=12, replace=False)
    pool_k = rng.choice(np.arange(1, 70000 if wide else 20000), size=n_k_values, replace=False)
    coords = set()
    if lattice:
        # every (b, m, n) collected at every k: one member class (the presets' shape)
        mn = set()
        while len(mn) * n_k_values < R:
            mn.add((int(rng.integers(1, 5)), int(rng.choice(pool_m)), int(rng.choice(pool_n))))
        coords = {(b, m, n, int(k)) for (b, m, n) in mn for k in pool_k}
    while len(coords) < R:
        coords.add((int(rng.integers(1, 5)), int(rng.choice(pool_m)), int(rng.choice(pool_n)),
                    int(rng.choice(pool_k))))
    coords = sorted(coords, key=lambda c: (c[1], c[2], c[3], c[0]))
    co = np.array(coords, np.uint64)
    cand = rng.integers(-1, C, size=R).astype(np.int64)   # some kernels without curves
    t = {"exact_coords": co, "exact_coords_curve": cand.copy(), "cand_curve": cand,
         "log_m": np.log2(co[:, 1].astype(np.float64)), "log_n": np.log2(co[:, 2].astype(np.float64)),
         "log_k": np.log2(co[:, 3].astype(np.float64))}
    import math
    for name, col in (("log_m", 1), ("log_n", 2), ("log_k", 3)):
        t[name] = np.array([math.log2(int(v)) for v in co[:, col]], np.float64)
    offs = [0]
    dims, thrs = [], []
    for c in range(C):
        ns = int(rng.integers(2, 12))
        d = np.sort(rng.choice(np.arange(1, 20000), size=ns, replace=False)).astype(np.float64)
        dims += list(d)
        thrs += list(rng.uniform(1.0, 900.0, ns))
        offs.append(len(dims))
    t.update(sample_offsets=np.array(offs, np.int64), sample_dims=np.array(dims),
             sample_thrs=np.array(thrs),
             ref_dim=np.array([dims[offs[c + 1] - 1] for c in range(C)]),
             ref_dur=rng.uniform(1.0, 500.0, C), ref_waves=rng.integers(1, 9, C).astype(np.float64),
             tile_m=rng.choice([16, 32, 64, 128, 256], C).astype(np.uint64),
             tile_n=rng.choice([16, 32, 64, 128, 256], C).astype(np.uint64),
             split_k=rng.choice([1, 1, 2, 4], C).astype(np.uint64),
             blocks_per_wave=rng.choice([30, 132, 148, 296], C).astype(np.uint64),
             family_rowblock=np.full(C, 1 if rowblock else 0, np.uint8))
    t["ref_thr"] = np.array([thrs[offs[c + 1] - 1] for c in range(C)])
    t["exact_keys"] = None
    return t, pool_m, pool_n, pool_k


@pytest.mark.parametrize("seed,R,C,nkv,rowblock,lattice", [
    (1, 40, 5, 3, False, False), (2, 300, 20, 40, False, False),
    (3, 900, 60, 120, False, False), (4, 200, 7, 9, True, False),
    (5, 64, 3, 64, False, False), (6, 1500, 30, 33, False, False),
    (7, 90, 6, 9, False, True), (8, 540, 60, 9, False, True), (9, 400, 12, 40, False, True),
    (10, 60, 4, 5, True, True)])
def test_random_tables_grid(gpu, seed, R, C, nkv, rowblock, lattice):
    import torch
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(seed)
    t, pm, pn, pk = random_tables(rng, R, C, nkv, rowblock, lattice=lattice)
    dt = _native.DeviceTables(t, 0)
    # axes mix recorded values (exact hits, exact distance ties) and others
    B = np.array(sorted({1, 2, 3, 4, 7}), np.uint64)
    M = np.array(sorted(set(rng.choice(pm, 5).tolist()) | set(rng.integers(1, 6000, 5).tolist())), np.uint64)
    N = np.array(sorted(set(rng.choice(pn, 5).tolist()) | set(rng.integers(1, 6000, 5).tolist())), np.uint64)
    K = np.array(sorted(set(rng.choice(pk, 30).tolist()) | set(rng.integers(1, 30000, 300).tolist())), np.uint64)
    plan = _native.GridPlan(dt, (B, M, N, K))
    n = plan.cardinality
    dev = torch.device("cuda")
    lat = torch.empty(n, dtype=torch.float64, device=dev)
    cur = torch.empty(n, dtype=torch.int32, device=dev)
    blk = torch.empty(n, dtype=torch.int64, device=dev)
    wav = torch.empty(n, dtype=torch.int64, device=dev)
    stats = torch.tensor([-1, 0, 0], dtype=torch.int64, device=dev)
    plan.launch(lat, cur, blk, wav, nan_stats=stats)
    o_lat, o_cur, o_blk, o_wav = oracle.grid(t, (B, M, N, K), use_coords=True)
    assert np.array_equal(lat.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
    assert np.array_equal(cur.cpu().numpy(), o_cur)
    assert np.array_equal(wav.cpu().numpy().view(np.uint64), o_wav)
    assert np.array_equal(blk.cpu().numpy().view(np.uint64), o_blk)
    fast = torch.empty(n, dtype=torch.float64, device=dev)
    stats2 = torch.tensor([-1, 0, 0], dtype=torch.int64, device=dev)
    plan.launch(fast, nan_stats=stats2)
    assert np.array_equal(fast.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
    nan = np.isnan(o_lat)
    for st in (stats, stats2):
        st = st.cpu().numpy()
        assert st[1] == nan.sum()
        first = int(np.argmax(nan)) if nan.any() else -1
        if st[2] == 0:
            assert st[0] == first
    # explicit-descriptor kernel on the same tables
    pts = np.array(np.meshgrid(B, M, N, K, indexing="ij")).reshape(4, -1).T.astype(np.uint32)
    sel = rng.choice(len(pts), min(len(pts), 5000), replace=False)
    shapes = np.ascontiguousarray(pts[sel])
    d_s = torch.from_numpy(shapes).to(dev)
    m = len(sel)
    outs = [torch.empty(m, dtype=dt_, device=dev) for dt_ in
            (torch.float64, torch.int32, torch.int32, torch.int8, torch.int32, torch.float64)]
    _native.check(_native.load().pm2l_points_predict(
        dt.handle, d_s.data_ptr(), m, *[o.data_ptr() for o in outs], _native.stream_handle()),
        "points")
    ref = oracle.points(t, shapes)
    got = [o.cpu().numpy() for o in outs]
    assert np.array_equal(got[0].view(np.uint64), ref[0].view(np.uint64))
    assert np.array_equal(got[1], ref[1])
    assert np.array_equal(got[3], ref[3])
    assert np.array_equal(got[4], ref[4])
    assert np.array_equal(got[5].view(np.uint64), ref[5].view(np.uint64))
    assert dt.groups == len(np.unique(t["log_k"]))


@pytest.mark.parametrize("seed,R,C,nkv,nb,nm", [
    (11, 540, 60, 9, 4, 40), (12, 90, 6, 9, 8, 36), (13, 400, 12, 40, 1, 12),
    (14, 200, 20, 20, 2, 30), (15, 60, 4, 5, 4, 40), (16, 300, 9, 3, 8, 35)])
def test_lookup_path_random_lattice(gpu, seed, R, C, nkv, nb, nm):
    """One-member-class tables (every (b, m, n) recorded at every k), an even
    k axis and full 1/2/4/8-value batch slabs: the one-class lookup kernel
    (kernel path 3) against the oracle, bit for bit, plus NaN statistics."""
    import torch
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(seed)
    t, pm, pn, pk = random_tables(rng, R, C, nkv, lattice=True)
    dt = _native.DeviceTables(t, 0)
    B = np.array([1, 2, 3, 4, 5, 7, 8, 9][:nb], np.uint64)
    h = nm // 2
    M = np.array(sorted(set(rng.choice(pm, h).tolist()) | set(rng.integers(1, 9000, nm - h).tolist())), np.uint64)
    N = np.array(sorted(set(rng.choice(pn, h).tolist()) | set(rng.integers(1, 9000, nm - h).tolist())), np.uint64)
    K = sorted(set(pk.tolist()) | set((pk + 1).tolist()) | set(rng.integers(1, 40000, 160).tolist()))
    K = np.array(K[:len(K) // 2 * 2], np.uint64)
    plan = _native.GridPlan(dt, (B, M, N, K))
    dev = torch.device("cuda")
    lat = torch.empty(plan.cardinality, dtype=torch.float64, device=dev)
    assert plan.kernel_path(lat) == 3
    stats = torch.tensor([-1, 0, 0], dtype=torch.int64, device=dev)
    plan.launch(lat, nan_stats=stats)
    o_lat, *_ = oracle.grid(t, (B, M, N, K), use_coords=True)
    got = lat.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), o_lat.view(np.uint64))
    nan = np.isnan(o_lat)
    st = stats.cpu().numpy()
    assert st[1] == nan.sum()
    if st[2] == 0:
        assert st[0] == (int(np.argmax(nan)) if nan.any() else -1)


def test_lookup_path_used_for_bench_grid(gpu):
    """The C2 bench grid runs on the lookup kernel."""
    import torch
    import bench
    from paper_2603_00549_b200 import _native
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import PreparedGrid
    ds = bench.load_bf16()
    prep = PreparedGrid(ds, bench.grid_for(1), WaveModel(ds.device.sm_count))
    plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
    lat = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    assert plan.kernel_path(lat) == 3
    assert plan.kernel_path(lat, verify=True) == 2


@pytest.mark.parametrize("seed,rowblock,lattice", [(21, True, False), (22, True, True), (23, False, False)])
def test_long_k_axis_few_rows_is_k_tiled(gpu, seed, rowblock, lattice):
    """Attention-shaped grids (m = n = 1, many batch values, a long k axis):
    the general grid kernel splits the k axis into tiles; bit-exact against
    the oracle, verify and latency-only launches alike."""
    import torch
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(seed)
    t, pm, pn, pk = random_tables(rng, 120, 8, 12, rowblock=rowblock, lattice=lattice)
    dt = _native.DeviceTables(t, 0)
    B = np.array([8, 12, 16, 24, 40, 64, 96], np.uint64)
    M = np.array([1], np.uint64) if rowblock else np.array([int(pm[0])], np.uint64)
    N = np.array([1], np.uint64) if rowblock else np.array([int(pn[0])], np.uint64)
    K = np.array(sorted(set(rng.integers(1, 60000, 6001).tolist()) | set(pk.tolist())), np.uint64)
    plan = _native.GridPlan(dt, (B, M, N, K))
    n = plan.cardinality
    dev = torch.device("cuda")
    lat = torch.empty(n, dtype=torch.float64, device=dev)
    cur = torch.empty(n, dtype=torch.int32, device=dev)
    blk = torch.empty(n, dtype=torch.int64, device=dev)
    wav = torch.empty(n, dtype=torch.int64, device=dev)
    plan.launch(lat, cur, blk, wav)
    o_lat, o_cur, o_blk, o_wav = oracle.grid(t, (B, M, N, K), use_coords=True)
    assert np.array_equal(lat.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
    assert np.array_equal(cur.cpu().numpy(), o_cur)
    assert np.array_equal(wav.cpu().numpy().view(np.uint64), o_wav)
    fast = torch.empty(n, dtype=torch.float64, device=dev)
    stats = torch.tensor([-1, 0, 0], dtype=torch.int64, device=dev)
    plan.launch(fast, nan_stats=stats)
    assert np.array_equal(fast.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
    nan = np.isnan(o_lat)
    st = stats.cpu().numpy()
    assert st[1] == nan.sum()
    if st[2] == 0:
        assert st[0] == (int(np.argmax(nan)) if nan.any() else -1)


@pytest.mark.parametrize("seed,nk", [(31, 6000), (32, 4096), (33, 2050)])
def test_lookup_path_long_k_chunks(gpu, seed, nk):
    """k axes longer than one 2048-k chunk: chunk-local ranks, per-k tables
    read from global memory (not staged), 64-byte map segments."""
    import torch
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(seed)
    t, pm, pn, pk = random_tables(rng, 360, 30, 9, lattice=True)
    dt = _native.DeviceTables(t, 0)
    B = np.array([1, 2, 4, 8], np.uint64)
    M = np.array(sorted(set(rng.choice(pm, 3).tolist()) | set(rng.integers(1, 9000, 3).tolist())), np.uint64)
    N = np.array(sorted(set(rng.choice(pn, 3).tolist()) | set(rng.integers(1, 9000, 2).tolist())), np.uint64)
    K = sorted(set(pk.tolist()) | set(rng.integers(1, 60000, 2 * nk).tolist()))
    K = np.array(K[:nk // 2 * 2], np.uint64)   # even length: pair stores
    assert len(K) > 2048 and len(K) % 2 == 0
    plan = _native.GridPlan(dt, (B, M, N, K))
    lat = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    assert plan.kernel_path(lat) == 3
    stats = torch.tensor([-1, 0, 0], dtype=torch.int64, device="cuda")
    plan.launch(lat, nan_stats=stats)
    o_lat, *_ = oracle.grid(t, (B, M, N, K), use_coords=True)
    assert np.array_equal(lat.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
    assert stats.cpu().numpy()[1] == np.isnan(o_lat).sum()


def test_misaligned_output_and_odd_k_axis(gpu):
    """A latency buffer that is not 16-byte aligned, or an odd k axis: the
    lookup kernel writes each pair with two 8-byte stores (and masks the
    last pair of an odd chunk); same bits as the oracle."""
    import torch
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(41)
    t, pm, pn, pk = random_tables(rng, 120, 12, 6, lattice=True)
    dt = _native.DeviceTables(t, 0)
    B = np.array([1, 2, 3, 4], np.uint64)
    M = np.array(sorted(set(rng.integers(1, 6000, 6).tolist())), np.uint64)
    N = np.array(sorted(set(rng.integers(1, 6000, 5).tolist())), np.uint64)
    for nk in (300, 301, 2049):
        K = np.array(sorted(set(rng.integers(1, 30000, 3 * nk).tolist()))[:nk], np.uint64)
        assert len(K) == nk
        plan = _native.GridPlan(dt, (B, M, N, K))
        buf = torch.empty(plan.cardinality + 1, dtype=torch.float64, device="cuda")
        aligned, shifted = buf[:plan.cardinality], buf[1:]
        assert plan.kernel_path(aligned) == 3 and plan.kernel_path(shifted) == 3
        o_lat, *_ = oracle.grid(t, (B, M, N, K), use_coords=True)
        for out in (aligned, shifted):
            stats = torch.tensor([-1, 0, 0], dtype=torch.int64, device="cuda")
            buf.fill_(-1.0)
            plan.launch(out, nan_stats=stats)
            assert np.array_equal(out.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
            assert stats.cpu().numpy()[1] == np.isnan(o_lat).sum()
        # nothing written outside the slice
        assert buf[-1].item() == -1.0 or buf[0].item() == -1.0


@pytest.mark.parametrize("seed,nk,nb,b_max", [(51, 1000, 4, 9000), (52, 4096, 8, 9000),
                                              (53, 2400, 2, 9000), (54, 1000, 4, 3_000_000)])
def test_lookup_path_row_block_tables(gpu, seed, nk, nb, b_max):
    """Row-block (attention / triton_vec) one-class tables take the lookup
    kernel with the per-point (b, k) wave model; bit-exact, NaN stats.
    b_max = 3e6 puts b*k past 32 bits: the two-step u64 wave count instead
    of the single tile_m * blocks_per_wave magic division."""
    import torch
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(seed)
    t, pm, pn, pk = random_tables(rng, 80, 6, 8, rowblock=True, lattice=True)
    dt = _native.DeviceTables(t, 0)
    B = np.array(sorted(set(rng.integers(1, b_max, 4 * nb).tolist()))[:nb], np.uint64)
    M = np.array([1], np.uint64)
    N = np.array([1], np.uint64)
    K = sorted(set(pk.tolist()) | set(rng.integers(1, 65000, 2 * nk).tolist()))
    K = np.array(K[:nk], np.uint64)
    assert len(K) == nk and nk % 2 == 0
    plan = _native.GridPlan(dt, (B, M, N, K))
    lat = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    assert plan.kernel_path(lat) == 3
    stats = torch.tensor([-1, 0, 0], dtype=torch.int64, device="cuda")
    plan.launch(lat, nan_stats=stats)
    o_lat, *_ = oracle.grid(t, (B, M, N, K), use_coords=True)
    assert np.array_equal(lat.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
    nan = np.isnan(o_lat)
    st = stats.cpu().numpy()
    assert st[1] == nan.sum()
    if st[2] == 0:
        assert st[0] == (int(np.argmax(nan)) if nan.any() else -1)


@pytest.mark.parametrize("seed,dup_batches", [(21, False), (22, True), (23, True)])
def test_points_one_class_exact_ties(gpu, seed, dup_batches):
    """Explicit descriptors on a one-class lattice whose coordinates are all
    powers of two, so every log2 is an exact integer and distances tie
    everywhere: the row-walk member search must return the reference's first
    index (lexicographic (distance, scan index) minimum), bit for bit against
    the oracle's linear scan.  Rows/columns are sparse (not a product set) and
    members repeat across batch values."""
    import math
    import torch
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(seed)
    pm = [2 ** e for e in range(3, 14)]
    pk = [2 ** e for e in range(4, 15, 2)]
    mn = set()
    while len(mn) < 40:
        mn.add((int(rng.integers(1, 4)) if dup_batches else 1, int(rng.choice(pm)), int(rng.choice(pm))))
    coords = sorted({(b, m, n, k) for (b, m, n) in mn for k in pk}, key=lambda c: (c[1], c[2], c[3], c[0]))
    co = np.array(coords, np.uint64)
    R, C = len(co), 7
    cand = rng.integers(0, C, size=R).astype(np.int64)
    t = {"exact_coords": co, "exact_coords_curve": cand.copy(), "cand_curve": cand, "exact_keys": None}
    for name, col in (("log_m", 1), ("log_n", 2), ("log_k", 3)):
        t[name] = np.array([math.log2(int(v)) for v in co[:, col]], np.float64)
    t.update(sample_offsets=np.arange(0, 2 * C + 1, 2, dtype=np.int64),
             sample_dims=np.tile([16.0, 20000.0], C), sample_thrs=rng.uniform(1, 900, 2 * C),
             ref_dim=np.full(C, 20000.0), ref_dur=rng.uniform(1, 500, C), ref_waves=np.ones(C),
             tile_m=np.full(C, 64, np.uint64), tile_n=np.full(C, 128, np.uint64),
             split_k=np.ones(C, np.uint64), blocks_per_wave=np.full(C, 148, np.uint64),
             family_rowblock=np.zeros(C, np.uint8))
    t["ref_thr"] = t["sample_thrs"][1::2].copy()
    dt = _native.DeviceTables(t, 0)
    q = [2 ** e for e in range(0, 17)] + [3 * 2 ** e for e in range(0, 12)]
    n = 60000
    shapes = np.stack([rng.integers(1, 5, n), rng.choice(q, n), rng.choice(q, n),
                       rng.choice(q + pk, n)], 1).astype(np.uint32)
    d_s = torch.from_numpy(shapes).cuda()
    outs = [torch.empty(n, dtype=dt_, device="cuda") for dt_ in
            (torch.float64, torch.int32, torch.int32, torch.int8, torch.int32, torch.float64)]
    _native.check(_native.load().pm2l_points_predict(
        dt.handle, d_s.data_ptr(), n, *[o.data_ptr() for o in outs], _native.stream_handle()),
        "points")
    ref = oracle.points(t, shapes)
    got = [o.cpu().numpy() for o in outs]
    assert np.array_equal(got[4], ref[4])       # record (first index on ties)
    assert np.array_equal(got[0].view(np.uint64), ref[0].view(np.uint64))
    assert np.array_equal(got[3], ref[3])
    assert np.array_equal(got[5].view(np.uint64), ref[5].view(np.uint64))


@pytest.mark.parametrize("seed,rowblock,ties", [(31, True, False), (32, True, True), (33, False, False),
                                                (34, False, True)])
def test_single_member_tables(gpu, seed, rowblock, ties):
    """Tables whose records all share one (m, n) (the attention / triton
    presets' shape): the planner-free single-member kernel (path 4) through
    the host plan and the device planner, against the oracle bit for bit --
    many-row grids, exact hits on several batch values, kernels without a
    curve (NaN + statistics) and, with ``ties``, k values equidistant from
    two k-groups (powers of two)."""
    import math
    import torch
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(seed)
    m0, n0 = (1, 1) if rowblock else (int(rng.integers(16, 512)), int(rng.integers(16, 512)))
    ks = sorted({2 ** int(e) for e in rng.integers(4, 16, 6)}) if ties else \
        sorted({int(x) for x in rng.integers(16, 40000, 7)})
    bs = [1, 3, 96]
    coords = sorted({(b, m0, n0, k) for b in bs for k in ks}, key=lambda c: (c[1], c[2], c[3], c[0]))
    co = np.array(coords, np.uint64)
    R, C = len(co), 5
    cand = rng.integers(-1, C, R).astype(np.int64)
    t = {"exact_coords": co, "exact_coords_curve": cand.copy(), "cand_curve": cand, "exact_keys": None}
    for name, col in (("log_m", 1), ("log_n", 2), ("log_k", 3)):
        t[name] = np.array([math.log2(int(v)) for v in co[:, col]], np.float64)
    offs = [0]
    dims, thrs = [], []
    for _ in range(C):
        d = np.sort(rng.choice(np.arange(1, 60000), 8, replace=False)).astype(np.float64)
        dims += list(d)
        thrs += list(rng.uniform(1.0, 900.0, 8))
        offs.append(len(dims))
    t.update(sample_offsets=np.array(offs, np.int64), sample_dims=np.array(dims),
             sample_thrs=np.array(thrs), ref_dim=np.array([dims[o - 1] for o in offs[1:]]),
             ref_dur=rng.uniform(1, 500, C), ref_waves=rng.integers(1, 5, C).astype(np.float64),
             tile_m=rng.choice([64, 128, 256], C).astype(np.uint64),
             tile_n=rng.choice([64, 128], C).astype(np.uint64),
             split_k=rng.choice([1, 2], C).astype(np.uint64),
             blocks_per_wave=rng.choice([30, 148, 296], C).astype(np.uint64),
             family_rowblock=np.full(C, 1 if rowblock else 0, np.uint8))
    t["ref_thr"] = np.array([thrs[o - 1] for o in offs[1:]])
    dt = _native.DeviceTables(t, 0)
    B = np.array(sorted(set(bs) | {2, 7, 500}), np.uint64)
    if rowblock:
        M = N = np.array([1], np.uint64)
    else:
        M = np.array(sorted({m0, 1, 5, 4000} | set(rng.integers(2, 3000, 4).tolist())), np.uint64)
        N = np.array(sorted({n0, 3, 7000} | set(rng.integers(2, 3000, 3).tolist())), np.uint64)
    K = np.array(sorted(set(ks) | {3 * k // 2 for k in ks} | set(rng.integers(1, 70000, 500).tolist())),
                 np.uint64)
    o_lat = oracle.grid(t, (B, M, N, K), use_coords=True, verify=False)
    nan = np.isnan(o_lat)
    # host plan
    plan = _native.GridPlan(dt, (B, M, N, K))
    lat = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    stats = torch.tensor([-1, 0, 0], dtype=torch.int64, device="cuda")
    assert plan.kernel_path(lat) == 4
    plan.launch(lat, nan_stats=stats)
    assert np.array_equal(lat.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
    st = stats.cpu().numpy()
    assert st[1] == nan.sum() and st[0] == (int(np.argmax(nan)) if nan.any() else -1)
    # device planner (device-resident axes)
    axes = [torch.from_numpy(a.view(np.int64)).cuda() for a in (B, M, N, K)]
    dp = _native.DeviceGridPlanner(dt, *(len(a) for a in axes))
    out = torch.full((plan.cardinality,), -1.0, dtype=torch.float64, device="cuda")
    dp.launch(axes, out, nan_stats=stats)
    assert dp.kernel_path() == 4 and dp.status() == 0
    assert np.array_equal(out.cpu().numpy().view(np.uint64), o_lat.view(np.uint64))
    # a batch sub-slice
    part = torch.empty((2 * len(M) * len(N) * len(K),), dtype=torch.float64, device="cuda")
    dp.launch(axes, part, b_lo=1, b_hi=3)
    inner = len(M) * len(N) * len(K)
    assert np.array_equal(part.cpu().numpy().view(np.uint64), o_lat[inner:3 * inner].view(np.uint64))
