#!/usr/bin/env python3
"""Small launches of every kernel of libpm2l_b200.so, for compute-sanitizer
(memcheck / racecheck / synccheck; tests/test_gpu_sanitizer.py):

  grid_ring_kernel (one-class lookup path, host plan and device planner,
  PAIR and odd k axes, row-block tables), grid_kernel (general path with
  the verification outputs), plan_kernel, base_table_kernel, fixup_kernel,
  all_curves_kernel, points_kernel (row walk, member pass, general sweep),
  points_curve_kernel, membound_kernel, segment_fsum_kernel,
  store_count/scan/encode_kernel, store_lookup_kernel, nan_scan,
  single_kernel (the flash-attention grid, exact hits at batch 96),
  grid_error_kernel, partition_cut_kernel / partition_best_kernel.
Every result is compared with the oracle so a sanitizer run also proves the
launches did their work.  Exit status 0 on success.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the checker)


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def main():
    from conftest import dataset
    from paper_2603_00549_b200 import _native, backend
    from paper_2603_00549_b200.aggregate import segment_fsum
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.membound import MemBoundModel, predict_membound_batch
    from paper_2603_00549_b200.nascache import (GridSpec, PreparedGrid, encode_records,
                                                encode_records_device)
    from test_gpu_random_tables import random_tables

    ds = dataset("bf16")
    gen = dataset("generic_bf16")
    wm = WaveModel(ds.device.sm_count)
    grids = [
        (ds, GridSpec("matmul", DType.BF16, TransposeMode.NN, {
            "batch": (1, 2, 3, 4), "m": (64, 100, 128, 1000), "n": (96, 128, 777),
            "k": tuple(range(16, 3000, 97)) + (4096,)})),
        (ds, GridSpec("linear", DType.BF16, TransposeMode.TN, {
            "batch": (1, 2), "m": (32, 300), "n": (64, 65), "k": tuple(range(32, 2000, 61))})),
        (gen, GridSpec("flash_attention", DType.BF16, TransposeMode.NN, {
            "batch": (8, 96, 640), "k": tuple(range(64, 5000, 37))})),
    ]
    for d, g in grids:
        prep = PreparedGrid(d, g, WaveModel(d.device.sm_count))
        want = oracle.grid(prep.tables(), prep.axis_arrays())
        lat, cur, blk, wav = (x.cpu().numpy() for x in backend.predict_grid_device(prep, verify=True))
        assert np.array_equal(bits(lat), bits(want[0])) and np.array_equal(cur, want[1])
        fast = backend.predict_grid_device(prep).cpu().numpy()     # lookup kernel / planner
        assert np.array_equal(bits(fast), bits(want[0]))
        plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
        out = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
        plan.launch(out)
        assert np.array_equal(bits(out.cpu().numpy()), bits(want[0]))
        plan.close()
        allc = backend.predict_grid_all_curves(prep)
        assert allc.shape[1] == g.cardinality
        recs = encode_records_device(g, backend.predict_grid_device(prep))
        assert recs.tobytes() == encode_records(g, want[0]).tobytes()
        assert backend.first_nan(backend.predict_grid_device(prep)) == -1
    # store writer + batched lookup (store_lookup_kernel)
    import tempfile
    from paper_2603_00549_b200.nascache import CacheStore, write_store
    g = grids[0][1]
    lat0 = backend.predict_grid(PreparedGrid(ds, g, wm))
    with tempfile.TemporaryDirectory() as tmp:
        path = os.path.join(tmp, "s.bin")
        write_store(path, g, ds, lat0)
        with CacheStore(path) as st:
            pts = list(g.iter_points())[::7]
            got = st.lookup_many(pts)
            assert np.array_equal(bits(got), bits(lat0[::7]))
    # explicit descriptors: one-class row walk (bf16), random lattice / general tables
    rng = np.random.default_rng(3)
    prep = PreparedGrid(ds, grids[0][1], wm)
    shapes = np.stack([rng.integers(1, 9, 3000), rng.integers(1, 5000, 3000),
                       rng.integers(1, 5000, 3000), rng.integers(1, 20000, 3000)], 1).astype(np.uint32)
    for t, dt in ((prep.tables(), prep.device_tables(0)),
                  *[(tt, _native.DeviceTables(tt, 0)) for tt in
                    (random_tables(rng, 300, 20, 40)[0], random_tables(rng, 90, 6, 9, lattice=True)[0],
                     random_tables(rng, 64, 3, 64)[0])]):
        s = torch.from_numpy(shapes).cuda()
        n = len(shapes)
        outs = [torch.empty(n, dtype=x, device="cuda") for x in
                (torch.float64, torch.int32, torch.int32, torch.int8, torch.int32, torch.float64)]
        _native.check(_native.load().pm2l_points_predict(
            dt.handle, s.data_ptr(), n, *[o.data_ptr() for o in outs], _native.stream_handle()),
            "points")
        ref = oracle.points(t, shapes)
        assert np.array_equal(bits(outs[0].cpu().numpy()), bits(ref[0]))
        cid = torch.from_numpy(rng.integers(0, len(t["sample_offsets"]) - 1, n).astype(np.int32)).cuda()
        lat = torch.empty(n, dtype=torch.float64, device="cuda")
        det = torch.empty((n, 4), dtype=torch.float64, device="cuda")
        _native.check(_native.load().pm2l_points_predict_curve(
            dt.handle, s.data_ptr(), cid.data_ptr(), n, lat.data_ptr(), 0, det.data_ptr(),
            _native.stream_handle()), "points_curve")
        want = oracle.points_curve(t, shapes, cid.cpu().numpy())[0]
        assert np.array_equal(bits(lat.cpu().numpy()), bits(want))
    # membound + exact sums
    models = [MemBoundModel("softmax", DType.FP32, (1e-9, 2e-9, 1e-10, 3e-10, 1e-11), 1.5, "d", 0, 0)]
    f = rng.uniform(0, 1e9, (1000, 5))
    lat, _ = predict_membound_batch(models, f, np.zeros(1000, np.int32))
    olat, _ = oracle.membound(f, np.zeros(1000, np.int32), np.array(models[0].weights),
                              np.array([1.5]), np.array([2.0]))
    assert np.array_equal(bits(lat), bits(olat))
    offs = np.array([0, 3, 3, 100, 1000], np.int64)
    assert np.array_equal(bits(segment_fsum(lat, offs)), bits(oracle.segment_fsum(lat, offs)))
    # §8f row 4: interpolation-grid audit and the partition cut scan
    from test_audit import AUDIT, _curve, _fixture, _fx, _truth
    from paper_2603_00549_b200.curvefit import grid_error_report
    from paper_2603_00549_b200.partition import partition_two_device
    for rep in AUDIT["grid_error"][:3]:
        r = grid_error_report(_curve(rep["kernel"]), _truth(rep), max_points=rep["max_points"])
        assert r.max_rel_err.hex() == _fx(rep["max_rel_err"]).hex()
    for p in AUDIT["partition"][:3]:
        graph, ds_a, ds_b = _fixture([_fx(x) for x in p["lat_a"]], [_fx(x) for x in p["lat_b"]])
        if not p["link"]:
            assert partition_two_device(graph, ds_a, ds_b).cut_after_layer_index == p["cut"]
    print("sanitize_smoke: ok")


if __name__ == "__main__":
    main()
