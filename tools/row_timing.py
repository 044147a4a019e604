#!/usr/bin/env python3
"""Per-phase timeline of the one-class lookup kernel (diagnostics).

Build the instrumented library here:   python tools/row_timing.py --build
Run on a B200:  PM2L_LIB_PATH=$PWD/paper_2603_00549_b200/libpm2l_timing.so python tools/row_timing.py

Each warp's lane 0 stamps %globaltimer at: 0 kernel entry, 1 tile start
(prologue done; SM clock64 cycles / SM_MHZ), 2 staircase, 3 W table, 4 cut searches, 5 byte maps,
6 base table visible, 7 tile written.
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2603_00549_b200", "libpm2l_timing.so")


def build():
    from paper_2603_00549_b200 import _build
    print(_build.build(extra_flags=["-DPM2L_TIMING"], out_path=LIB))


def main():
    import ctypes as C
    import numpy as np
    import torch
    import bench
    from paper_2603_00549_b200 import _native
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import PreparedGrid
    lib = _native.load()
    fn = lib.pm2l_debug_row_timing
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int]
    if os.environ.get("ROW_TIMING_GRID") == "c3":  # attention grid of tools/profile_c3.py
        from paper_2603_00549_b200 import load_dataset
        from paper_2603_00549_b200.core import DType, TransposeMode
        from paper_2603_00549_b200.nascache import GridSpec
        ds = load_dataset(os.path.join(ROOT, "tests", "golden", "datasets", "generic_bf16.json"))
        bh = sorted({b * h for b in (1, 2, 4, 8, 16, 32, 64, 128) for h in (8, 12, 16, 20, 32, 40, 64)})
        grid = GridSpec("cutlass_attention", DType.BF16, TransposeMode.NN,
                        {"batch": tuple(bh), "m": (1,), "n": (1,), "k": tuple(range(64, 65536))})
    else:
        ds = bench.load_bf16()
        grid = bench.grid_for(1)
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    mode = os.environ.get("ROW_TIMING_PLAN", "host")   # host | dplan (step) | dplan2 (grid alone)
    if mode == "host":
        plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
        out = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
        print("kernel path", plan.kernel_path(out))
        run = lambda: plan.launch(out, stages=7)  # noqa: E731
    else:
        axes = [torch.from_numpy(np.ascontiguousarray(a, np.uint64).view(np.int64)).cuda()
                for a in prep.axis_arrays()]
        dp = _native.DeviceGridPlanner(prep.device_tables(0), *(len(a) for a in axes))
        out = torch.empty(grid.cardinality, dtype=torch.float64, device="cuda")
        dp.launch(axes, out)
        print("kernel path", dp.kernel_path())
        if mode == "dplan":
            run = lambda: dp.launch(axes, out)  # noqa: E731
        else:
            def run():
                dp.launch(axes, out, stages=1)
                torch.cuda.synchronize()
                dp.launch(axes, out, stages=2)
    for _ in range(5):
        flush.zero_()
        ev[0].record()
        run()
        ev[1].record()
    torch.cuda.synchronize()
    print("step ms (last)", ev[0].elapsed_time(ev[1]))
    n = 16384 * 8
    buf = np.zeros(n, np.uint64)
    assert fn(buf.ctypes.data, n) == 0
    tiles = int(os.environ.get("ROW_TILES", "2500"))
    t = buf[:tiles * 8].reshape(tiles, 8).astype(np.int64)
    # entry stamp is per (cta, warp) == tile index for a one-tile-per-warp launch
    # SM clock64 stamps: per-tile differences only (clocks differ across SMs)
    mhz = float(os.environ.get("SM_MHZ", "1965"))
    rel = (t - t[:, :1]) / mhz
    if os.environ.get("PM2L_ROW_RING", "1") != "0":
        # ring kernel: 0 CTA entry, 1 build start, 2 build end, 3 emit start, 4 emit end
        names = ["entry", "build start", "build end", "emit start", "emit end"]
        for i in range(1, 5):
            print(f"{names[i]:<12} (from CTA entry) median {np.median(rel[:, i]):6.2f}  "
                  f"p10 {np.percentile(rel[:, i], 10):6.2f}  p90 {np.percentile(rel[:, i], 90):6.2f}  max {rel[:, i].max():6.2f}")
        # static CTA-strided tiles: tile = cta + j * ctas
        ctas = int(os.environ.get("RING_CTAS", "444"))
        cta_end = np.array([rel[c::ctas, 4].max() for c in range(ctas)])
        cta_n = np.array([len(rel[c::ctas]) for c in range(ctas)])
        for nt in sorted(set(cta_n.tolist())):
            e = cta_end[cta_n == nt]
            print(f"CTAs with {nt} tiles: {len(e)}, end median {np.median(e):.2f} p90 {np.percentile(e, 90):.2f} max {e.max():.2f}")
        pd = np.zeros(4096 * 4, np.uint64)
        assert fn(pd.ctypes.data, -len(pd)) == 0
        pd = pd.reshape(-1, 4)[:ctas].astype(np.int64)
        pr = (pd - pd[:, :1]) / mhz
        print(f"writers (CTA entry=0): reach pdl wait median {np.median(pr[:, 1]):.2f}, leave "
              f"median {np.median(pr[:, 2]):.2f} max {pr[:, 2].max():.2f}, first FULL median "
              f"{np.median(pr[:, 3]):.2f} max {pr[:, 3].max():.2f} us")
        d = lambda a, b: np.median(rel[:, b] - rel[:, a])  # noqa: E731
        print(f"build: staircase {d(1, 5):.2f}  W {d(5, 6):.2f}  cuts {d(6, 7):.2f}  maps {d(7, 2):.2f}")
        print("build dur median", np.median(rel[:, 2] - rel[:, 1]), " emit dur median",
              np.median(rel[:, 4] - rel[:, 3]), " wait full median", np.median(rel[:, 3] - rel[:, 2]))
        return
    names = ["entry", "prologue", "staircase", "W table", "cuts", "maps", "pdl wait", "emit"]
    print("phase            median_us   p90_us   max_us")
    for i in range(1, 8):
        d = rel[:, i] - rel[:, i - 1]
        print(f"{names[i]:<15} {np.median(d):9.2f} {np.percentile(d, 90):8.2f} {d.max():8.2f}")
    print("tile span us: median", np.median(rel[:, 7]), "max", rel[:, 7].max())


if __name__ == "__main__":
    if "--build" in sys.argv:
        build()
    else:
        main()
