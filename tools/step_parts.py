#!/usr/bin/env python3
"""Composition of one bench step: CUDA-graph replays of growing prefixes of
the step (stats reset, base table, grid kernel, fix-ups), L2 flushed before
each, CUDA events around the replay."""
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
    ds = bench.load_bf16()
    prep = PreparedGrid(ds, bench.grid_for(1), WaveModel(ds.device.sm_count))
    plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
    dev = torch.device("cuda")
    outs = [torch.empty(plan.cardinality, dtype=torch.float64, device=dev) for _ in range(4)]
    out = outs[0]
    stats = torch.empty(3, dtype=torch.int64, device=dev)
    init = torch.tensor([-1, 0, 0], dtype=torch.int64, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    out = outs[0]
    variants = {
        "empty": lambda: None,
        "reset": lambda: stats.copy_(init),
        "base": lambda: plan.launch(out, nan_stats=stats, stages=1),
        "base+grid": lambda: plan.launch(out, nan_stats=stats, stages=3),
        "grid only": lambda: plan.launch(out, nan_stats=stats, stages=2),
        "fixup only": lambda: plan.launch(out, nan_stats=stats, stages=4),
        "all": lambda: plan.launch(out, nan_stats=stats, stages=7),
        "reset+all": lambda: (stats.copy_(init), plan.launch(out, nan_stats=stats, stages=7)),
    }
    for _ in range(3):
        plan.launch(out, nan_stats=stats, stages=7)
    torch.cuda.synchronize()
    print("fixups", plan.n_fixups)
    for mode in ("flushed", "rotating"):
        print("--", mode)
        for name, fn in variants.items():
            gs = []
            for o in outs:
                out = o
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    fn()
                gs.append(g)
            ts = []
            for i in range(16):
                if mode == "flushed":
                    flush.zero_()
                if name == "grid only":   # base table hot, as inside a step
                    plan.launch(outs[i % 4], nan_stats=stats, stages=1)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                gs[i % 4 if mode == "rotating" else 0].replay()
                e1.record()
                if mode == "flushed":
                    torch.cuda.synchronize()
                if i >= 4:
                    ts.append((e0, e1))
            torch.cuda.synchronize()
            ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ts)
            print(f"{name:<12} median {ts[len(ts)//2]:7.1f} us   min {ts[0]:7.1f} us")


if __name__ == "__main__":
    main()
