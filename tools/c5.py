#!/usr/bin/env python3
"""BASELINE configs[4] / SURVEY §8d C5 on ONE B200: rank 0's shard of the
1 B-point mixed NAS precompute over 8 GPUs.  Each GEMM/attention grid is
split into 8 contiguous batch slabs (paper_2603_00549_b200.shard); this
runs slab 0 of every component (device-resident output, CUDA events,
256 MiB L2 flush before each component) plus 1/8 of the membound vectors.

    matmul BF16 NN   8 x 100 x 100 x 7500   (600 M)
    linear BF16 TN   8 x  50 x 100 x 5000   (200 M)
    bmm    BF16 NN   8 x  50 x  50 x 5000   (100 M)
    flash + cutlass attention BF16: 600 batch' x 62500 seq (37.5 M each)
    membound         25 M feature vectors
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_00549_b200 import _native, load_dataset  # noqa: E402
from paper_2603_00549_b200.compute import WaveModel  # noqa: E402
from paper_2603_00549_b200.core import DType, TransposeMode  # noqa: E402
from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid  # noqa: E402
from paper_2603_00549_b200.shard import shard_bounds  # noqa: E402

WORLD = 8
B8 = (1, 2, 4, 8, 16, 32, 64, 128)


def gemm(family, tmode, nm, nn, kstep, nk):
    return GridSpec(family, DType.BF16, tmode, {
        "batch": B8, "m": tuple(range(64, 64 + 61 * nm, 61)), "n": tuple(range(96, 96 + 53 * nn, 53)),
        "k": tuple(range(32, 32 + kstep * nk, kstep))})


def attention(family):
    return GridSpec(family, DType.BF16, TransposeMode.NN, {
        "batch": tuple(range(8, 8 + 8 * 600, 8)), "m": (1,), "n": (1,),
        "k": tuple(range(64, 64 + 62500))})


def run_grid(name, ds, grid, flush):
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    lo, hi = shard_bounds(len(grid.axes["batch"]), WORLD, 0)
    plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays(), lo, hi)
    out = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    stats = torch.empty(3, dtype=torch.int64, device="cuda")
    for _ in range(2):
        plan.launch(out, nan_stats=stats)
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.launch(out, nan_stats=stats)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = float(np.median(ts))
    return {"component": name, "points": plan.cardinality, "s": t, "pred_per_s": plan.cardinality / t,
            "kernel_path": plan.kernel_path(out), "unresolved": int(stats[1].item())}


def run_membound(n, flush):
    rng = np.random.default_rng(23)
    nm = 32
    f = torch.from_numpy(rng.uniform(0, 1e9, (n, 5))).cuda()
    ids = torch.from_numpy(rng.integers(0, nm, n).astype(np.int32)).cuda()
    w = torch.from_numpy(rng.normal(size=(nm, 5)) * 1e-8).cuda()
    b = torch.from_numpy(rng.uniform(0, 3, nm)).cuda()
    fl = torch.full((nm,), 2.0, dtype=torch.float64, device="cuda")
    lat = torch.empty(n, dtype=torch.float64, device="cuda")
    flo = torch.empty(n, dtype=torch.uint8, device="cuda")
    lib = _native.load()
    call = lambda: _native.check(lib.pm2l_membound_predict(  # noqa: E731
        f.data_ptr(), ids.data_ptr(), n, w.data_ptr(), b.data_ptr(), fl.data_ptr(), nm,
        lat.data_ptr(), flo.data_ptr(), _native.stream_handle()), "membound")
    call()
    ts = []
    for _ in range(5):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        call()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3)
    t = float(np.median(ts))
    return {"component": "membound", "points": n, "s": t, "pred_per_s": n / t}


def main():
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    bf16 = load_dataset(os.path.join(ROOT, "tests", "golden", "datasets", "bf16.json"))
    gen = load_dataset(os.path.join(ROOT, "tests", "golden", "datasets", "generic_bf16.json"))
    rows = [
        run_grid("matmul bf16 NN", bf16, gemm("matmul", TransposeMode.NN, 100, 100, 8, 7500), flush),
        run_grid("linear bf16 TN", bf16, gemm("linear", TransposeMode.TN, 50, 100, 12, 5000), flush),
        run_grid("bmm bf16 NN", bf16, gemm("batched_matmul", TransposeMode.NN, 50, 50, 12, 5000), flush),
        run_grid("flash_attention bf16", gen, attention("flash_attention"), flush),
        run_grid("cutlass_attention bf16", gen, attention("cutlass_attention"), flush),
        run_membound(25_000_000 // WORLD, flush),
    ]
    for r in rows:
        print(json.dumps(r))
    pts = sum(r["points"] for r in rows)
    t = sum(r["s"] for r in rows)
    print(json.dumps({"C5 rank-0 shard": pts, "s": t, "pred_per_s_per_gpu": pts / t,
                      "projected_8gpu_pred_per_s": WORLD * pts / t,
                      "note": "weak-scaling projection: shards are independent (no data-path collective)"}))


if __name__ == "__main__":
    main()
