#!/usr/bin/env python3
"""Launch the C2 grid plan a few times (for ncu / nsight captures).

    ncu --set full -k regex:grid_kernel -s 2 -c 1 -o gpurun_out/prof python tools/profile_grid.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_00549_b200 import _native  # noqa: E402
from paper_2603_00549_b200.compute import WaveModel  # noqa: E402
from paper_2603_00549_b200.nascache import PreparedGrid  # noqa: E402


def main():
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 5
    ds = bench.load_bf16()
    prep = PreparedGrid(ds, bench.grid_for(1), WaveModel(ds.device.sm_count))
    plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
    out = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    for _ in range(reps):
        plan.launch(out)
    torch.cuda.synchronize()
    print("ok", plan.cardinality, float(out[:4].sum()))


if __name__ == "__main__":
    main()
