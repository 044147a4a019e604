#!/usr/bin/env python3
"""Host cost of the small device calls predict_model is made of (warm,
per call, microseconds): ctypes launches, torch allocations / copies."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_00549_b200 import _native  # noqa: E402
from paper_2603_00549_b200.membound import MemBoundModel  # noqa: E402
from paper_2603_00549_b200.core import DType  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / n * 1e6


lib = _native.load()
dev = torch.device("cuda")
f = torch.rand(5, dtype=torch.float64, device=dev)
ids = torch.zeros(1, dtype=torch.int32, device=dev)
w = torch.rand(5, dtype=torch.float64, device=dev)
b = torch.zeros(1, dtype=torch.float64, device=dev)
fl = torch.zeros(1, dtype=torch.float64, device=dev)
o = torch.empty(1, dtype=torch.float64, device=dev)
fo = torch.empty(1, dtype=torch.uint8, device=dev)
s = _native.stream_handle()
r = {}
r["pm2l_membound_predict (1 op)"] = per_call(lambda: lib.pm2l_membound_predict(
    f.data_ptr(), ids.data_ptr(), 1, w.data_ptr(), b.data_ptr(), fl.data_ptr(), 1, o.data_ptr(),
    fo.data_ptr(), s))
r["stream_handle()"] = per_call(lambda: _native.stream_handle())
r["torch.empty(8) cuda"] = per_call(lambda: torch.empty(8, dtype=torch.float64, device=dev))
x = np.zeros(40, np.float64)
r["H2D 320 B (from_numpy().to)"] = per_call(lambda: torch.from_numpy(x).to(dev))
y = torch.zeros(40, dtype=torch.float64, device=dev)
r["D2H 320 B (.cpu())"] = per_call(lambda: y.cpu())
r["cudaGetDeviceCount via pm2l_device_count"] = per_call(lambda: lib.pm2l_device_count())
print(json.dumps({k: round(v, 2) for k, v in r.items()}, indent=1))
