#!/usr/bin/env python3
"""Event-timed grid kernel and step: CUDA-graph replay vs direct stream
launches (both enqueued behind the 256 MiB flush kernel)."""
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
    ds = bench.load_bf16()
    prep = PreparedGrid(ds, bench.grid_for(1), WaveModel(ds.device.sm_count))
    plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
    out = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    stats = torch.empty(3, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    gs = {}
    for name, st in (("base", 1), ("grid", 2), ("step", 7)):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            plan.launch(out, nan_stats=stats, stages=st)
        gs[name] = g
    for _ in range(3):
        plan.launch(out, nan_stats=stats)
    torch.cuda.synchronize()

    def run(kind, what, reps=20):
        ts = []
        for _ in range(reps):
            flush.zero_()
            if what == "grid":
                gs["base"].replay() if kind == "graph" else plan.launch(out, nan_stats=stats, stages=1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if kind == "graph":
                gs[what].replay()
            else:
                plan.launch(out, nan_stats=stats, stages=2 if what == "grid" else 7)
            e1.record()
            ts.append((e0, e1))
        torch.cuda.synchronize()
        v = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
        return np.median(v), v[0]

    for what in ("grid", "step"):
        for kind in ("graph", "direct"):
            med, mn = run(kind, what)
            print(f"{what:<5} {kind:<7} median {med:6.2f} us  min {mn:6.2f} us")


if __name__ == "__main__":
    main()
