"""GPU edge cases from the round-1 review: axis orders the raw FFI accepts,
signed per-model sums, and the Prediction invariant of the array model API."""

import math

import numpy as np
import pytest

import oracle
from conftest import dataset, ffi_slice, golden_meta, prepared

pytestmark = pytest.mark.gpu

GRIDS = {g["name"]: g for g in golden_meta()["grids"]}


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.mark.parametrize("name", ["matmul_bf16", "exact_mix_bf16", "cutlass_attn_bf16"])
def test_shuffled_k_axis_through_ffi_slice(gpu, name):
    """The reference's predict_grid_slice takes axes in any order; the lookup
    kernel's byte maps assume an ascending k axis, so a shuffled one must take
    the order-independent path and still equal the oracle / compiled
    reference point for point."""
    from paper_2603_00549_b200 import _native
    prep = prepared(GRIDS[name])
    t = dict(prep.tables())
    B, M, N, K = prep.axis_arrays()
    rng = np.random.default_rng(17)
    for Ks in (K[::-1].copy(), K[rng.permutation(len(K))].copy()):
        axes = (B, M, N, Ks)
        out = np.empty(len(B) * len(M) * len(N) * len(Ks), np.float64)
        ffi_slice(t, axes, 0, len(B), out)
        want = oracle.grid(t, axes, 0, len(B), verify=False)
        assert np.array_equal(_bits(out), _bits(want))
        mod = oracle.reference_kernels()
        if mod is not None:
            ref = oracle.reference_predict_grid(mod, t, axes, jobs=2)
            assert np.array_equal(_bits(out), _bits(ref))
        plan = _native.GridPlan(prep.device_tables(0), axes)
        import torch
        probe = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
        if len(Ks) > 1:
            assert plan.kernel_path(probe) != 3, "lookup kernel on an unsorted k axis"
        plan.close()


def test_advice_example_descending_k_two_groups(gpu):
    """k = [8192, 16] against k-groups {16, 8192}: k = 16 must resolve to
    the group at log2 k = 4."""
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid
    ds = dataset("bf16")
    grid = GridSpec("matmul", DType.BF16, TransposeMode.NN,
                    {"batch": (1, 2), "m": (100, 3000), "n": (96, 700), "k": (16, 8192)})
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    t = dict(prep.tables())
    B, M, N, K = prep.axis_arrays()
    axes = (B, M, N, K[::-1].copy())
    out = np.empty(8 * 2, np.float64)
    ffi_slice(t, axes, 0, 2, out)
    assert np.array_equal(_bits(out), _bits(oracle.grid(t, axes, 0, 2, verify=False)))


def test_segment_fsum_signed_terms(gpu):
    """math.fsum semantics for segments with negative terms, exact
    cancellation, +-inf and NaN (negative terms gave NaN)."""
    from paper_2603_00549_b200.aggregate import segment_fsum
    rng = np.random.default_rng(23)
    lens = rng.integers(1, 80, 2000)
    offs = np.concatenate([[0], np.cumsum(lens)])
    v = rng.uniform(-1e4, 1e4, offs[-1]) * 10.0 ** rng.integers(-8, 9, offs[-1])
    v[offs[3]:offs[4]] = np.concatenate([[1e20, 1.0, -1e20]] + [[0.5]] * (lens[3] - 3))[:lens[3]]
    v[offs[5]] = 1e300                       # dynamic range beyond the window
    v[offs[6]:offs[7]] = -(2.0 ** -1000)
    got = segment_fsum(v, offs)
    want = np.array([math.fsum(v[offs[i]:offs[i + 1]]) for i in range(len(lens))])
    assert np.array_equal(_bits(got), _bits(want))
    # exact cancellation -> +0.0; halfway cases with mixed signs
    v = np.array([1.0, -1.0, 3.5, -3.5, -0.0, 1.0, -(2.0 ** -53), 2.0 ** -106,
                  -1.0, 2.0 ** -53, -(2.0 ** -106)])
    o = np.array([0, 2, 5, 8, 11])
    want = [math.fsum(v[o[i]:o[i + 1]]) for i in range(4)]
    assert np.array_equal(_bits(segment_fsum(v, o)), _bits(np.array(want)))
    inf = np.inf
    v = np.array([inf, 1.0, -inf, 2.0, inf, -inf, np.nan, 1.0])
    o = np.array([0, 2, 4, 6, 8])
    got = segment_fsum(v, o)
    assert got[0] == inf and got[1] == -inf and np.isnan(got[2]) and np.isnan(got[3])


def test_model_grid_rejects_nonpositive_layer(gpu):
    """A raw membound layer below a non-positive floor is not a valid
    Prediction in the reference (core.py:383-386); the array API raises the
    same ValidationError instead of summing it."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tools"))
    import c4
    from paper_2603_00549_b200.aggregate import TemplateLayer, predict_model_grid
    from paper_2603_00549_b200.core import DType
    from paper_2603_00549_b200.errors import ValidationError
    ds = dataset("fp32_full")
    params = [(1, 64, 256, 2), (2, 128, 512, 4)]
    fams = ("linear", "linear", "linear", "batched_matmul", "utility:softmax", "linear", "linear",
            "linear")
    template = [TemplateLayer(i, f, DType.FP32) for i, f in zip(c4.TEMPLATE_IDS, fams)]
    shapes, feats = c4.grid_arrays(params)
    lat, tot = predict_model_grid(template, shapes, feats, ds)
    assert (lat > 0).all()
    feats = np.array(feats, np.float64)
    feats[:, 4, :] = 0.0                      # softmax raw = intercept
    try:
        predict_model_grid(template, shapes, feats, ds, membound_floor_us=-math.inf)
    except ValidationError:
        pass  # negative intercept: rejected like the reference
    else:
        lat2, tot2 = predict_model_grid(template, shapes, feats, ds, membound_floor_us=-math.inf)
        assert (lat2 > 0).all()
        for i in range(len(params)):
            assert tot2[i] == math.fsum(lat2[i])


@pytest.mark.parametrize("name", ["matmul_bf16", "exact_mix_bf16", "cutlass_attn_bf16"])
def test_empty_single_and_partial_slices_through_ffi_slice(gpu, name):
    """Slice bounds as the reference's callers pass them (_kernels.pyx:76-90,
    backend.py:64-76): an empty batch slice writes nothing, a one-point grid
    and a partial batch slice equal the oracle point for point."""
    prep = prepared(GRIDS[name])
    t = dict(prep.tables())
    B, M, N, K = prep.axis_arrays()
    # empty slice: nothing written
    out = np.full(4, 7.0)
    ffi_slice(t, (B, M, N, K), 1, 1, out)
    assert np.all(out == 7.0)
    # one point
    axes1 = (B[:1].copy(), M[-1:].copy(), N[:1].copy(), K[len(K) // 2:len(K) // 2 + 1].copy())
    out1 = np.empty(1, np.float64)
    ffi_slice(t, axes1, 0, 1, out1)
    assert np.array_equal(_bits(out1), _bits(oracle.grid(t, axes1, 0, 1, verify=False)))
    # a partial slice of the batch axis: the slice's points, in slice order
    if len(B) > 1:
        lo, hi = 1, len(B)
        outp = np.empty((hi - lo) * len(M) * len(N) * len(K), np.float64)
        ffi_slice(t, (B, M, N, K), lo, hi, outp)
        want = oracle.grid(t, (B, M, N, K), lo, hi, verify=False)
        assert np.array_equal(_bits(outp), _bits(want))


@pytest.mark.parametrize("name", ["matmul_bf16", "exact_mix_bf16"])
def test_repeated_and_shuffled_axis_values_through_ffi_slice(gpu, name):
    """The reference loops over whatever axis arrays it is given: repeated
    values and shuffled m / n / batch axes must give the oracle's points."""
    prep = prepared(GRIDS[name])
    t = dict(prep.tables())
    B, M, N, K = prep.axis_arrays()
    rng = np.random.default_rng(5)
    cases = [
        (B, M, N, np.repeat(K[:7], 2)),                                   # repeated k
        (np.repeat(B[:2], 2), M[rng.permutation(len(M))].copy(), N, K),  # repeated b, shuffled m
        (B[::-1].copy(), M, N[rng.permutation(len(N))].copy(), K),       # reversed b, shuffled n
    ]
    for axes in cases:
        axes = tuple(np.ascontiguousarray(a, np.uint64) for a in axes)
        n = len(axes[0]) * len(axes[1]) * len(axes[2]) * len(axes[3])
        out = np.empty(n, np.float64)
        ffi_slice(t, axes, 0, len(axes[0]), out)
        want = oracle.grid(t, axes, 0, len(axes[0]), verify=False)
        assert np.array_equal(_bits(out), _bits(want))


def test_points_empty_batch_and_invalid_coordinates(gpu):
    """Explicit descriptors: an empty batch is a no-op; a zero coordinate is
    an invalid op (NaN latency, curve -1), as the reference's resolver
    refuses non-positive shapes (core.py validation)."""
    import torch
    from paper_2603_00549_b200 import _native
    prep = prepared(GRIDS["matmul_bf16"])
    dt = prep.device_tables(0)
    lib = _native.load()
    lat = torch.full((4,), 7.0, dtype=torch.float64, device="cuda")
    cur = torch.full((4,), 9, dtype=torch.int32, device="cuda")
    wav = torch.zeros(4, dtype=torch.int32, device="cuda")
    shapes = torch.tensor([[1, 128, 128, 64], [0, 128, 128, 64], [1, 0, 128, 64], [1, 128, 128, 0]],
                          dtype=torch.int32, device="cuda")
    _native.check(lib.pm2l_points_predict(dt.handle, shapes.data_ptr(), 0, lat.data_ptr(),
                                          cur.data_ptr(), wav.data_ptr(), 0, 0, 0,
                                          _native.stream_handle()), "points n=0")
    torch.cuda.synchronize()
    assert torch.all(lat == 7.0) and torch.all(cur == 9)
    _native.check(lib.pm2l_points_predict(dt.handle, shapes.data_ptr(), 4, lat.data_ptr(),
                                          cur.data_ptr(), wav.data_ptr(), 0, 0, 0,
                                          _native.stream_handle()), "points")
    torch.cuda.synchronize()
    l, c = lat.cpu().numpy(), cur.cpu().numpy()
    assert math.isfinite(l[0]) and c[0] >= 0
    assert np.all(np.isnan(l[1:])) and np.all(c[1:] == -1)


def test_ffi_slice_is_thread_safe(gpu):
    """pm2l_predict_grid_slice is documented synchronous and thread-safe
    (include/pm2l.h): concurrent callers (ctypes drops the GIL) on different
    tables and slices each get their own bit-exact result."""
    import threading
    names = ["matmul_bf16", "exact_mix_bf16", "cutlass_attn_bf16", "parity_fp32", "wide_fp32"]
    names = [n for n in names if n in GRIDS]
    jobs = []
    for name in names:
        prep = prepared(GRIDS[name])
        t = dict(prep.tables())
        axes = prep.axis_arrays()
        n = len(axes[0]) * len(axes[1]) * len(axes[2]) * len(axes[3])
        jobs.append((t, axes, oracle.grid(t, axes, 0, len(axes[0]), verify=False), n))
    errors = []

    def run(t, axes, want, n):
        try:
            for _ in range(5):
                out = np.empty(n, np.float64)
                ffi_slice(t, axes, 0, len(axes[0]), out)
                if not np.array_equal(_bits(out), _bits(want)):
                    errors.append("mismatch")
        except Exception as exc:  # surfaced below
            errors.append(repr(exc))

    threads = [threading.Thread(target=run, args=j) for j in jobs for _ in range(2)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors[:3]
