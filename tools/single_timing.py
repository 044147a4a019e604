#!/usr/bin/env python3
"""Per-CTA timeline of the single-(m, n) grid kernel (diagnostics).

Build here:     python tools/row_timing.py --build
Run on a B200:  PM2L_LIB_PATH=$PWD/paper_2603_00549_b200/libpm2l_timing.so python tools/single_timing.py
Prints CTA entry / staged / first item resolved / exit (globaltimer, us)
for the C3 grid after an L2 flush.
"""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2603_00549_b200 import _native, load_dataset
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid
    lib = _native.load()
    fn = lib.pm2l_debug_row_timing
    fn.restype = C.c_int
    fn.argtypes = [C.c_void_p, C.c_int]
    ds = load_dataset(os.path.join(ROOT, "tests", "golden", "datasets", "generic_bf16.json"))
    bh = sorted({b * h for b in (1, 2, 4, 8, 16, 32, 64, 128) for h in (8, 12, 16, 20, 32, 40, 64)})
    grid = GridSpec(os.environ.get("FAMILY", "flash_attention"), DType.BF16, TransposeMode.NN,
                    {"batch": tuple(bh), "m": (1,), "n": (1,), "k": tuple(range(64, 65536))})
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    plan = _native.GridPlan(prep.device_tables(0), prep.axis_arrays())
    out = torch.empty(plan.cardinality, dtype=torch.float64, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    print("kernel path", plan.kernel_path(out))
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    for _ in range(4):
        flush.zero_()
        ev[0].record()
        plan.launch(out)
        ev[1].record()
    torch.cuda.synchronize()
    print("call ms (last)", ev[0].elapsed_time(ev[1]))
    n = 4096 * 4
    buf = np.zeros(n, np.uint64)
    assert fn(buf.ctypes.data, -n) == 0
    ctas = int(os.environ.get("CTAS", "256"))
    v = buf.reshape(-1, 4)[:ctas].astype(np.int64)
    t0 = v[:, 0].min()
    r = (v - t0) / 1e3
    for i, name in enumerate(["entry", "staged", "first item", "exit"]):
        print(f"{name:<11} median {np.median(r[:, i]):7.2f}  p10 {np.percentile(r[:, i], 10):7.2f}  "
              f"p90 {np.percentile(r[:, i], 90):7.2f}  max {r[:, i].max():7.2f} us")
    slow = np.argsort(-r[:, 3])[:8]
    print("slowest CTAs:", [(int(c), round(float(r[c, 3]), 2), round(float(r[c, 2]), 2)) for c in slow])


if __name__ == "__main__":
    main()
