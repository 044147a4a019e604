#!/usr/bin/env python3
"""Launch the C3 attention grid (cutlass_attention BF16) a few times (ncu)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2603_00549_b200 import _native, load_dataset  # noqa: E402
from paper_2603_00549_b200.compute import WaveModel  # noqa: E402
from paper_2603_00549_b200.core import DType, TransposeMode  # noqa: E402
from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid  # noqa: E402

ds = load_dataset(os.path.join(ROOT, "tests", "golden", "datasets", "generic_bf16.json"))
bh = sorted({b * h for b in (1, 2, 4, 8, 16, 32, 64, 128) for h in (8, 12, 16, 20, 32, 40, 64)})
grid = GridSpec("cutlass_attention", DType.BF16, TransposeMode.NN,
                {"batch": tuple(bh), "m": (1,), "n": (1,), "k": tuple(range(64, 65536))})
prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
out = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 4):
    plan.launch(out)
torch.cuda.synchronize()
print("ok", plan.cardinality)
