#!/usr/bin/env python3
"""Secondary throughput lines for the other SURVEY §8 rows (device-resident
inputs, CUDA events after warm-up, 256 MiB L2 flush before each timed run):

  C3      flash / cutlass attention grid (BF16): 28 B*H batch values x
          seq 64..65535 (row-block families, general grid kernel)
  points  C2 shapes as explicit 16-byte descriptors (exact + nearest
          resolution, tile/wave model, interpolation) -- pm2l_points_predict
  modeX   every (shape, candidate kernel) pair -- pm2l_grid_predict_all_curves
  membound  25 M feature vectors -- pm2l_membound_predict
Prints one JSON object per mode.
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_00549_b200 import _native, load_dataset  # noqa: E402
from paper_2603_00549_b200.compute import WaveModel  # noqa: E402
from paper_2603_00549_b200.core import DType, TransposeMode  # noqa: E402
from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid  # noqa: E402

FLUSH = None


def timed(fn, reps=10):
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    ts = []
    for _ in range(reps):
        FLUSH.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    return float(np.median(ts))


def c3(family):
    ds = load_dataset(os.path.join(ROOT, "tests", "golden", "datasets", "generic_bf16.json"))
    bh = sorted({b * h for b in (1, 2, 4, 8, 16, 32, 64, 128) for h in (8, 12, 16, 20, 32, 40, 64)})
    grid = GridSpec(family, DType.BF16, TransposeMode.NN,
                    {"batch": tuple(bh), "m": (1,), "n": (1,), "k": tuple(range(64, 65536))})
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
    out = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    t_replay = timed(lambda: plan.launch(out))
    # plan-inclusive: the device planner + grid kernel per call, axes in HBM
    axes = [torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).cuda()
            for a in prep.axis_arrays()]
    dp = _native.DeviceGridPlanner(prep.device_tables(0), *(len(a) for a in axes))
    t = timed(lambda: dp.launch(axes, out))
    return {"mode": f"C3 {family} bf16", "points": plan.cardinality, "s": t,
            "pred_per_s": plan.cardinality / t, "kernel_path": dp.kernel_path(),
            "plan": "device planner inside the timed call",
            "replayed_host_plan_pred_per_s": plan.cardinality / t_replay,
            "GB_per_s_written": 8 * plan.cardinality / t / 1e9}


def points():
    ds = bench.load_bf16()
    grid = bench.grid_for(1)
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    rng = np.random.default_rng(0)
    n = 10_000_000
    idx = rng.integers(0, grid.cardinality, n)
    pts = np.stack(np.unravel_index(idx, grid.shape()), 1)
    shapes = np.stack([np.asarray(grid.axes[a], np.uint32)[pts[:, i]]
                       for i, a in enumerate(("batch", "m", "n", "k"))], 1)
    s = torch.from_numpy(np.ascontiguousarray(shapes)).cuda()
    lat = torch.empty(n, dtype=torch.float64, device="cuda")
    cur = torch.empty(n, dtype=torch.int32, device="cuda")
    wav = torch.empty(n, dtype=torch.int32, device="cuda")
    dt = prep.device_tables(0)
    lib = _native.load()
    t = timed(lambda: _native.check(lib.pm2l_points_predict(
        dt.handle, s.data_ptr(), n, lat.data_ptr(), cur.data_ptr(), wav.data_ptr(), 0, 0, 0,
        _native.stream_handle()), "points"))
    return {"mode": "points (explicit descriptors, C2 shapes, bf16 tables)", "points": n, "s": t,
            "pred_per_s": n / t, "GB_per_s": 32 * n / t / 1e9,
            "bytes_per_pred": "16 in + 8 lat + 4 curve + 4 waves"}


def mode_x():
    ds = bench.load_bf16()
    g = bench.grid_for(1)
    axes = dict(g.axes)
    axes["m"] = axes["m"][:10]   # 4 x 10 x 50 x 1000 = 2 M shapes x 60 kernels
    grid = GridSpec(g.family, g.dtype, g.transpose_mode, axes)
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    from paper_2603_00549_b200 import backend
    out = backend.predict_grid_all_curves(prep)
    n = out.numel()
    t = timed(lambda: backend.predict_grid_all_curves(prep))
    return {"mode": "mode X (every shape x every candidate kernel)", "pairs": n, "s": t,
            "pred_per_s": n / t, "GB_per_s_written": 8 * n / t / 1e9}


def membound():
    from paper_2603_00549_b200.membound import MemBoundModel
    rng = np.random.default_rng(1)
    n, nm = 25_000_000, 32
    f = torch.from_numpy(rng.uniform(0, 1e9, (n, 5))).cuda()
    ids = torch.from_numpy(rng.integers(0, nm, n).astype(np.int32)).cuda()
    w = torch.from_numpy(rng.normal(size=(nm, 5)) * 1e-8).cuda()
    b = torch.from_numpy(rng.uniform(0, 3, nm)).cuda()
    fl = torch.full((nm,), 2.0, dtype=torch.float64, device="cuda")
    lat = torch.empty(n, dtype=torch.float64, device="cuda")
    flo = torch.empty(n, dtype=torch.uint8, device="cuda")
    lib = _native.load()
    t = timed(lambda: _native.check(lib.pm2l_membound_predict(
        f.data_ptr(), ids.data_ptr(), n, w.data_ptr(), b.data_ptr(), fl.data_ptr(), nm,
        lat.data_ptr(), flo.data_ptr(), _native.stream_handle()), "membound"))
    return {"mode": "membound (5-feature linear model + floor)", "ops": n, "s": t,
            "pred_per_s": n / t, "GB_per_s": 53 * n / t / 1e9, "bytes_per_pred": "40 + 4 in, 8 + 1 out"}


if __name__ == "__main__":
    modes = {"c3": [lambda: c3("cutlass_attention"), lambda: c3("flash_attention")],
             "points": [points], "modex": [mode_x], "membound": [membound]}
    pick = sys.argv[1:] or list(modes)
    for m in pick:
        for fn in modes[m]:
            print(json.dumps(fn()), flush=True)
