"""Device-side planner (plan.cu) against the host planner (tables.cpp
build_grid) and the oracle: the same latencies / curve ids / blocks / waves,
the same unresolved-point statistics, the same fix-up count and kernel path,
for every golden grid, randomised tables (ties, NaN curves, exact hits, many
k-groups, long k axes) and the full-size C2 grid; axis-contract violations
are reported in the sticky status word."""

import numpy as np
import pytest
import torch

import oracle
from conftest import golden_meta, prepared
from test_gpu_random_tables import random_tables

pytestmark = pytest.mark.gpu

GRIDS = {g["name"]: g for g in golden_meta()["grids"]}
LUT_N = 1 << 22


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def _dev_axes(axes):
    return [torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).cuda() for a in axes]


def _canonical(axes):
    return all(len(a) >= 1 and np.all(np.diff(a.astype(np.int64)) > 0) and a.min() >= 1
               for a in axes) and all(a.max() < LUT_N for a in axes[1:])


def host_vs_device(dt, axes, b_lo=0, b_hi=None, verify=True):
    """Run one slice through the host plan and the device plan; assert equal
    outputs and statistics; return the device latencies (numpy)."""
    from paper_2603_00549_b200 import _native
    b_hi = len(axes[0]) if b_hi is None else b_hi
    plan = _native.GridPlan(dt, axes, b_lo, b_hi)
    dp = _native.DeviceGridPlanner(dt, *(len(a) for a in axes))
    d_axes = _dev_axes(axes)
    n = plan.cardinality
    dev = torch.device("cuda")
    res = {}
    for name, run in (("host", lambda *o, **kw: plan.launch(*o, **kw)),
                      ("dev", lambda *o, **kw: dp.launch(d_axes, *o, b_lo=b_lo, b_hi=b_hi, **kw))):
        lat = torch.full((n,), -1.0, dtype=torch.float64, device=dev)
        stats = torch.zeros(3, dtype=torch.int64, device=dev)
        run(lat, nan_stats=stats)
        out = {"lat": lat.cpu().numpy(), "stats": stats.cpu().numpy()}
        if verify:
            v = [torch.empty(n, dtype=t, device=dev) for t in (torch.float64, torch.int32,
                                                                 torch.int64, torch.int64)]
            run(v[0], curve=v[1], blocks=v[2], waves=v[3])
            out.update(vlat=v[0].cpu().numpy(), curve=v[1].cpu().numpy(),
                       blocks=v[2].cpu().numpy(), waves=v[3].cpu().numpy())
        res[name] = out
    torch.cuda.synchronize()
    h, d = res["host"], res["dev"]
    assert np.array_equal(_bits(d["lat"]), _bits(h["lat"]))
    # count and first-NaN (unless a fix-up dirtied it: both then flag [2])
    assert d["stats"][1] == h["stats"][1] and d["stats"][2] == h["stats"][2]
    if not h["stats"][2]:
        assert d["stats"][0] == h["stats"][0]
    if verify:
        for k in ("curve", "blocks", "waves"):
            assert np.array_equal(d[k], h[k]), k
        assert np.array_equal(_bits(d["vlat"]), _bits(h["vlat"]))
    assert dp.status() == 0
    probe = torch.empty(n, dtype=torch.float64, device=dev)
    dp.launch(d_axes, probe, b_lo=b_lo, b_hi=b_hi)
    assert dp.kernel_path() == plan.kernel_path(probe)
    if dp.kernel_path() != 4:   # the single-member kernel runs no planner (no fix-up list)
        assert dp.fixups() == plan.n_fixups
    plan.close()
    dp.close()
    return d["lat"]


@pytest.mark.parametrize("name", list(GRIDS))
def test_device_plan_matches_host_plan_golden_grids(gpu, name):
    prep = prepared(GRIDS[name])
    axes = prep.axis_arrays()
    if not _canonical(axes):
        pytest.skip("axis values beyond the device planner's log2 table")
    lat = host_vs_device(prep.device_tables(0), axes)
    want = oracle.grid(prep.tables(), axes, verify=False)
    assert np.array_equal(_bits(lat), _bits(want))
    nb = len(axes[0])
    if nb > 1:
        host_vs_device(prep.device_tables(0), axes, 1, nb, verify=False)


@pytest.mark.parametrize("seed,R,C,nkv,rowblock,lattice,nk", [
    (1, 40, 5, 3, False, False, 300), (2, 300, 20, 40, False, False, 700),
    (3, 900, 60, 120, False, False, 2500), (4, 200, 7, 9, True, False, 400),
    (6, 1500, 30, 33, False, False, 5000), (7, 90, 6, 9, False, True, 800),
    (8, 540, 60, 9, False, True, 4097), (10, 60, 4, 5, True, True, 2048)])
def test_device_plan_random_tables(gpu, seed, R, C, nkv, rowblock, lattice, nk):
    from paper_2603_00549_b200 import _native
    rng = np.random.default_rng(seed)
    t, pm, pn, pk = random_tables(rng, R, C, nkv, rowblock, lattice=lattice)
    dt = _native.DeviceTables(t, 0)
    B = np.array([1, 2, 3, 4, 7, 8], np.uint64)
    M = np.array(sorted(set(rng.choice(pm, 5).tolist()) | set(rng.integers(1, 6000, 5).tolist())), np.uint64)
    N = np.array(sorted(set(rng.choice(pn, 5).tolist()) | set(rng.integers(1, 6000, 5).tolist())), np.uint64)
    K = np.array(sorted(set(rng.choice(pk, min(30, len(pk))).tolist())
                        | set(rng.integers(1, 60000, nk).tolist())), np.uint64)
    if len(K) % 2:
        K = K[:-1]
    axes = (B, M, N, K)
    lat = host_vs_device(dt, axes)
    want = oracle.grid(t, axes, verify=False)
    assert np.array_equal(_bits(lat), _bits(want))
    host_vs_device(dt, axes, 2, 5, verify=False)


def test_device_plan_full_c2_grid(gpu):
    """BASELINE configs[1] at full size (10M points): device plan == host plan."""
    import bench
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import PreparedGrid
    ds = bench.load_bf16()
    prep = PreparedGrid(ds, bench.grid_for(1), WaveModel(ds.device.sm_count))
    host_vs_device(prep.device_tables(0), prep.axis_arrays(), verify=False)


def test_device_plan_status_flags(gpu):
    from paper_2603_00549_b200 import _native
    prep = prepared(GRIDS["matmul_bf16"])
    dt = prep.device_tables(0)
    B, M, N, K = prep.axis_arrays()
    dp = _native.DeviceGridPlanner(dt, len(B), len(M) + 1, len(N), len(K))
    out = torch.empty(len(B) * (len(M) + 1) * len(N) * len(K), dtype=torch.float64, device="cuda")
    dp.launch(_dev_axes((B, M, N, K)), out)
    assert dp.status() == 0
    dp.launch(_dev_axes((B, M, N, K[::-1].copy())), out)
    assert dp.status() & 2
    assert dp.status() == 0          # sticky bits clear on read
    bad = np.concatenate([M, [np.uint64(LUT_N)]])
    dp.launch(_dev_axes((B, bad, N, K)), out)
    assert dp.status() & 1
    zero = M.copy()
    zero[0] = 0
    dp.launch(_dev_axes((B, zero, N, K)), out)
    assert dp.status() & 1
    # beyond the capacity: refused on the host
    from paper_2603_00549_b200.errors import ValidationError
    with pytest.raises(ValidationError):
        dp.launch(_dev_axes((B, M, N, np.arange(1, len(K) + 3, dtype=np.uint64))), out)
    dp.close()


def test_device_plan_is_graph_capturable(gpu):
    """One CUDA graph per step (planner + grid kernel), replayed with new axis
    contents in place: every replay plans the slice it finds."""
    from paper_2603_00549_b200 import _native
    prep = prepared(GRIDS["matmul_bf16"])
    dt = prep.device_tables(0)
    B, M, N, K = prep.axis_arrays()
    d_axes = _dev_axes((B, M, N, K))
    dp = _native.DeviceGridPlanner(dt, len(B), len(M), len(N), len(K))
    out = torch.empty(len(B) * len(M) * len(N) * len(K), dtype=torch.float64, device="cuda")
    stats = torch.zeros(3, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        dp.launch(d_axes, out, nan_stats=stats, stream=s)   # warm (lazy attributes)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        dp.launch(d_axes, out, nan_stats=stats, stream=s)
    for shift in (0, 7, 100):
        K2 = K + np.uint64(shift)
        d_axes[3].copy_(torch.from_numpy(K2.view(np.int64)))
        g.replay()
        torch.cuda.synchronize()
        want = oracle.grid(prep.tables(), (B, M, N, K2), verify=False)
        assert np.array_equal(_bits(out.cpu().numpy()), _bits(want))
    dp.close()
