#!/usr/bin/env python3
"""cProfile of warm single predict_model calls (host-side cost breakdown)."""
import cProfile
import json
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2603_00549_b200 as p  # noqa: E402
from paper_2603_00549_b200.aggregate import predict_model  # noqa: E402
from paper_2603_00549_b200.ingest import model_graph_from_json_obj  # noqa: E402

with open(os.path.join(ROOT, "tests", "golden", "models.json")) as fh:
    gold = json.load(fh)
ds = p.load_dataset(os.path.join(ROOT, "tests", "golden", "datasets", f"{gold['dataset']}.json"))
g = model_graph_from_json_obj(gold["models"][0]["graph"])
for _ in range(20):
    predict_model(g, ds)
pr = cProfile.Profile()
pr.enable()
for _ in range(200):
    predict_model(g, ds)
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(30)
