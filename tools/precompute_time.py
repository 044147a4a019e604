#!/usr/bin/env python3
"""nascache.precompute on the C2 grid (10 M points): prediction, device
record encoding + D2H, store file write; against the host encoder."""
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2603_00549_b200 import backend, nascache  # noqa: E402
from paper_2603_00549_b200.compute import WaveModel  # noqa: E402


def main():
    ds = bench.load_bf16()
    grid = bench.grid_for(1)
    wm = WaveModel(ds.device.sm_count)
    d = tempfile.mkdtemp()
    for rep in range(3):
        t0 = time.perf_counter()
        s = nascache.precompute(grid, ds, wm, os.path.join(d, "a.bin"))
        t1 = time.perf_counter()
        print(f"precompute (device encoder): {1e3 * (t1 - t0):.1f} ms total, predict {1e3 * s.elapsed_s:.2f} ms, "
              f"{grid.cardinality / (t1 - t0) / 1e6:.1f} M records/s")
    prep = nascache.PreparedGrid(ds, grid, wm)
    lat = backend.predict_grid_device(prep)
    for rep in range(2):
        t0 = time.perf_counter()
        rec = nascache.encode_records_device(grid, lat)
        t1 = time.perf_counter()
        host = lat.cpu().numpy()
        t2 = time.perf_counter()
        rec2 = nascache.encode_records(grid, host)
        t3 = time.perf_counter()
        print(f"encode: device+D2H {1e3 * (t1 - t0):.1f} ms, host numpy {1e3 * (t3 - t2):.1f} ms "
              f"(+{1e3 * (t2 - t1):.1f} ms D2H of latencies), equal={rec.tobytes() == rec2.tobytes()}")


if __name__ == "__main__" and "--lookups" not in sys.argv:
    main()


def lookups():
    import numpy as np
    ds = bench.load_bf16()
    grid = bench.grid_for(1)
    d = tempfile.mkdtemp()
    path = os.path.join(d, "c2.bin")
    nascache.precompute(grid, ds, WaveModel(ds.device.sm_count), path)
    rng = np.random.default_rng(0)
    with nascache.CacheStore(path) as st:
        idx = rng.integers(0, grid.cardinality, 4_000_000)
        pts = np.stack(np.unravel_index(idx, grid.shape()), 1)
        q = np.stack([np.asarray(grid.axes[a], np.uint64)[pts[:, i]]
                      for i, a in enumerate(nascache.AXIS_ORDER)], 1)
        st.lookup_many(q[:10])  # stage the records
        for rep in range(3):
            t0 = time.perf_counter()
            v = st.lookup_many(q)
            t1 = time.perf_counter()
            print(f"lookup_many: {len(q)} points in {1e3 * (t1 - t0):.1f} ms = {len(q) / (t1 - t0) / 1e6:.1f} M lookups/s (incl. H2D/D2H)")
        t0 = time.perf_counter()
        for p in q[:20000]:
            st.lookup(*(int(x) for x in p))
        t1 = time.perf_counter()
        print(f"scalar lookup (host mmap bsearch, reference algorithm): {20000 / (t1 - t0) / 1e3:.1f} k lookups/s")
        assert not np.isnan(v).any()


if __name__ == "__main__" and "--lookups" in sys.argv:
    lookups()
