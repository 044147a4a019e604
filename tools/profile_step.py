#!/usr/bin/env python3
"""The bench step (device planner + grid kernel on the C2 slice) a few
times, L2 flushed before each, for ncu captures of either kernel.

    ncu --set full -k regex:plan_kernel -s 2 -c 1 -o gpurun_out/plan python tools/profile_step.py
    ncu --set full -k regex:grid_ -s 2 -c 1 -o gpurun_out/grid python tools/profile_step.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_00549_b200 import _native  # noqa: E402
from paper_2603_00549_b200.compute import WaveModel  # noqa: E402
from paper_2603_00549_b200.nascache import PreparedGrid  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    ds = bench.load_bf16()
    prep = PreparedGrid(ds, bench.grid_for(1), WaveModel(ds.device.sm_count))
    axes = [torch.from_numpy(a.view(np.int64)).cuda() for a in bench.slice_axes(1, 0)]
    dp = _native.DeviceGridPlanner(prep.device_tables(0), *(len(a) for a in axes))
    n = int(np.prod([len(a) for a in axes]))
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    stats = torch.empty(3, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(reps):
        flush.zero_()
        dp.launch(axes, out, nan_stats=stats)
    torch.cuda.synchronize()
    print("ok", n, dp.kernel_path(), dp.status())


if __name__ == "__main__":
    main()
