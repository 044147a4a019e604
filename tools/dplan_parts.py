#!/usr/bin/env python3
"""Event-timed parts of the bench step, device plan vs host plan (diagnostics)."""
import os
import statistics
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
    dt = prep.device_tables(0)
    axes = [torch.from_numpy(a.view(np.int64)).cuda() for a in bench.slice_axes(1, 0)]
    dp = _native.DeviceGridPlanner(dt, *(len(a) for a in axes))
    hp = _native.GridPlan(dt, prep.axis_arrays())
    n = hp.cardinality
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    stats = torch.empty(3, dtype=torch.int64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    graphs = {}
    for name, fn in (("d_all", lambda: dp.launch(axes, out, nan_stats=stats)),
                     ("d_plan", lambda: dp.launch(axes, out, nan_stats=stats, stages=1)),
                     ("d_grid", lambda: dp.launch(axes, out, nan_stats=stats, stages=2)),
                     ("h_all", lambda: hp.launch(out, nan_stats=stats)),
                     ("h_base", lambda: hp.launch(out, nan_stats=stats, stages=1)),
                     ("h_grid", lambda: hp.launch(out, nan_stats=stats, stages=2))):
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
        graphs[name] = g
    torch.cuda.synchronize()
    s = torch.cuda.current_stream()

    def timed(seq, flush_first=True, reps=20):
        # seq: list of graph names; the LAST one is timed, the others run before
        res = []
        for _ in range(reps):
            if flush_first:
                flush.zero_()
            for nm in seq[:-1]:
                graphs[nm].replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            graphs[seq[-1]].replay()
            e1.record(s)
            torch.cuda.synchronize()
            res.append(e0.elapsed_time(e1) * 1e3)
        return statistics.median(res)

    for seq in (["d_all"], ["h_all"], ["d_plan"], ["h_base"], ["d_plan", "d_grid"],
                ["h_base", "h_grid"], ["d_grid"], ["h_grid"], ["h_base", "d_grid"],
                ["d_plan", "h_grid"]):
        print(f"{'+'.join(seq):16s} flushed {timed(seq):7.2f} us   warm {timed(seq, False):7.2f} us")


if __name__ == "__main__":
    main()
