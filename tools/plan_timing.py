#!/usr/bin/env python3
"""Per-role timeline of the device planner (diagnostics).

Build here:     python tools/plan_timing.py --build
Run on a B200:  PM2L_LIB_PATH=$PWD/paper_2603_00549_b200/libpm2l_timing.so python tools/plan_timing.py

Prints, per planner CTA role, entry / exit (globaltimer, us from the first
CTA's entry) of the C2 bench slice after an L2 flush.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_2603_00549_b200", "libpm2l_timing.so")


def main():
    if "--build" in sys.argv:
        from paper_2603_00549_b200 import _build
        print(_build.build(extra_flags=["-DPM2L_TIMING"], out_path=LIB))
        return
    import numpy as np
    import torch
    import bench
    from paper_2603_00549_b200 import _native
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.nascache import PreparedGrid
    lib = _native.load()
    fn = lib.pm2l_debug_plan_timing
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int]
    ds = bench.load_bf16()
    prep = PreparedGrid(ds, bench.grid_for(1), WaveModel(ds.device.sm_count))
    axes = [torch.from_numpy(a.view(np.int64)).cuda() for a in bench.slice_axes(1, 0)]
    dp = _native.DeviceGridPlanner(prep.device_tables(0), *(len(a) for a in axes))
    n = int(np.prod([len(a) for a in axes]))
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    nK = len(axes[3])
    nkc = (nK + 2047) // 2048
    kparts = (min(nK, 2048) + 15) // 16
    nrec = (prep.device_tables(0).n_records + 255) // 256
    nrow = (len(axes[1]) * len(axes[2]) + 255) // 256
    C_ = prep.device_tables(0).n_curves
    nblk = nkc * kparts + nrec + nrow + 1 + C_ * ((nK + 1023) // 1024)
    for rep in range(6):
        if rep < 3:
            flush.zero_()   # reps 3..5: warm L2 (code and tables cached)
        dp.launch(axes, out, stages=1)
        torch.cuda.synchronize()
        buf = (C.c_ulonglong * (8 * nblk))()
        fn(buf, 8 * nblk)
        v = np.array(buf, dtype=np.int64).reshape(-1, 8)
        t0 = v[:, 0].min()
        a0 = nkc * kparts
        roles = {"k-rank": v[:a0], "records": v[a0:a0 + nrec], "rows": v[a0 + nrec:a0 + nrec + nrow],
                 "m/n": v[a0 + nrec + nrow:a0 + nrec + nrow + 1], "base": v[a0 + nrec + nrow + 1:]}
        print(f"rep {rep}: " + "  ".join(
            f"{k}: {1e-3 * (r[:, 0].min() - t0):.2f}-{1e-3 * (r[:, 7].max() - t0):.2f}us"
            for k, r in roles.items()))
        for k in ("k-rank",):
            r = roles[k][0]
            print("   ", k, "phases (us):", [round(1e-3 * (x - t0), 2) for x in r if x > 0])


if __name__ == "__main__":
    main()
