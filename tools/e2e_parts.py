#!/usr/bin/env python3
"""Where the reference-FFI drop-in's time goes (C2 grid): the whole call,
the host plan build alone, a pinned 80 MB D2H, and host copies."""
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_00549_b200 import _native  # noqa: E402
from paper_2603_00549_b200.compute import WaveModel  # noqa: E402
from paper_2603_00549_b200.nascache import PreparedGrid  # noqa: E402


def tmin(fn, n=5):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts), 1e3 * sorted(ts)[len(ts) // 2]


def main():
    ds = bench.load_bf16()
    prep = PreparedGrid(ds, bench.grid_for(1), WaveModel(ds.device.sm_count))
    dev = torch.device("cuda")
    n = prep.grid.cardinality
    e2e = bench.run_e2e(prep, 0, 4, n, 5, 1, dev)
    print("e2e call ms", e2e["ms_per_step"], "G/s", e2e["value"] / 1e9)
    dt = prep.device_tables(0)
    axes = prep.axis_arrays()
    print("plan create (host build + H2D) ms min/med", tmin(lambda: _native.GridPlan(dt, axes).close()))
    d = torch.empty(n, dtype=torch.float64, device=dev)
    pin = torch.empty(n, dtype=torch.float64, pin_memory=True)
    page = np.empty(n, np.float64)
    page.fill(0)

    def d2h_pinned():
        pin.copy_(d, non_blocking=True)
        torch.cuda.synchronize()

    def d2h_page():
        page[:] = d.cpu().numpy()

    print("D2H pinned 80MB ms", tmin(d2h_pinned))
    print("D2H pageable (torch .cpu) ms", tmin(d2h_page))
    src = pin.numpy()
    for nt in (1, 4, 8, 16):
        def hcopy():
            ch = (n + nt - 1) // nt
            th = [threading.Thread(target=np.copyto, args=(page[i * ch:(i + 1) * ch], src[i * ch:(i + 1) * ch]))
                  for i in range(nt)]
            for t in th:
                t.start()
            for t in th:
                t.join()
        print(f"host copy pinned->pageable 80MB, {nt} threads ms", tmin(hcopy))
    print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))


if __name__ == "__main__":
    main()
