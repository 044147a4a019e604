#!/usr/bin/env python3
"""Drop-in API costs next to the reference's, on the same box:

  predict_grid   backend.predict_grid(prep) on the C2 grid (10 M points):
                 the Python plug-in point, pageable numpy result as the
                 reference's backend.py:61 allocates it; host time per call
                 (table staging cached after the first call, the kernel, the
                 80 MB device->host drain).  Reference: its backend.predict_grid
                 with the Cython kernel and jobs = host cores (baseline/_ref).
  predict_model  one predict_model(graph, dataset) call (TRANSFORMER_BLOCK,
                 tests/test_ingest.py:168-190 of the reference, via
                 tests/golden/models.json) -- single-call latency, warm.
                 Reference: its pure-Python predict_model (aggregate.py:173-196).
Prints one JSON object per line.
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

REF = os.path.join(ROOT, "baseline", "_ref")
DS = os.path.join(ROOT, "tests", "golden", "datasets")


def best(fn, reps):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return min(ts), float(np.median(ts))


def c2_axes():
    return {"batch": (1, 2, 4, 8), "m": tuple(range(64, 64 + 61 * 50, 61)),
            "n": tuple(range(96, 96 + 53 * 50, 53)), "k": tuple(range(32, 32 + 17 * 1000, 17))}


def ours():
    import paper_2603_00549_b200 as p
    from paper_2603_00549_b200 import backend
    from paper_2603_00549_b200.aggregate import predict_model
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.ingest import model_graph_from_json_obj
    ds = p.load_dataset(os.path.join(DS, "bf16.json"))
    grid = p.GridSpec("matmul", p.DType.BF16, p.TransposeMode.NN, c2_axes())
    prep = p.PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    b, med = best(lambda: backend.predict_grid(prep), 10)
    print(json.dumps({"api": "backend.predict_grid (C2, pageable numpy out)", "impl": "b200",
                      "best_s": b, "median_s": med, "pred_per_s": grid.cardinality / b}), flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "models.json")) as fh:
        gold = json.load(fh)
    full = p.load_dataset(os.path.join(DS, f"{gold['dataset']}.json"))
    g = model_graph_from_json_obj(gold["models"][0]["graph"])
    r = predict_model(g, full)
    assert r.total_latency_us.hex() == gold["models"][0]["total_hex"]
    b, med = best(lambda: predict_model(g, full), 200)
    print(json.dumps({"api": "predict_model (TRANSFORMER_BLOCK, %d layers)" % len(g.layers),
                      "impl": "b200", "best_s": b, "median_s": med,
                      "layers_per_s": len(g.layers) / med}), flush=True)


def reference():
    if not os.path.isdir(os.path.join(REF, "pm2lat")):
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref not installed"}))
        return
    sys.path.insert(0, REF)
    import pm2lat
    from pm2lat import backend
    from pm2lat.aggregate import predict_model
    from pm2lat.compute import WaveModel
    from pm2lat.core import DType, TransposeMode
    from pm2lat.ingest import load_dataset, model_graph_from_json_obj
    from pm2lat.nascache import GridSpec, PreparedGrid
    cores = len(os.sched_getaffinity(0))
    ds = load_dataset(os.path.join(DS, "bf16.json"))
    grid = GridSpec("matmul", DType.BF16, TransposeMode.NN, c2_axes())
    prep = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count))
    assert backend.active_backend() == "cython"
    b, med = best(lambda: backend.predict_grid(prep, jobs=cores), 1)
    print(json.dumps({"api": "backend.predict_grid (C2, pageable numpy out)",
                      "impl": "reference cython", "jobs": cores, "best_s": b, "median_s": med,
                      "pred_per_s": grid.cardinality / b,
                      "note": "the reference threads only the 4 batch values"}), flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "models.json")) as fh:
        gold = json.load(fh)
    full = load_dataset(os.path.join(DS, f"{gold['dataset']}.json"))
    g = model_graph_from_json_obj(gold["models"][0]["graph"])
    b, med = best(lambda: predict_model(g, full), 50)
    print(json.dumps({"api": "predict_model (TRANSFORMER_BLOCK, %d layers)" % len(g.layers),
                      "impl": "reference python", "best_s": b, "median_s": med,
                      "layers_per_s": len(g.layers) / med}), flush=True)
    _ = pm2lat


if __name__ == "__main__":
    which = sys.argv[1:] or ["ours", "reference"]
    if "ours" in which:
        ours()
    if "reference" in which:
        reference()
