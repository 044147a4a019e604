#!/usr/bin/env python3
"""BASELINE configs[3] / SURVEY §8d C4: whole-model latency over a NAS grid
of transformer blocks (TRANSFORMER_BLOCK template: q, k, v, out, up, down as
linear TN, scores as batched matmul, softmax as a memory-bound utility),
batch in {1..256} x seq in {64..8192} (powers of 2, batch*seq < 65536) x
14 hidden sizes x 3 MLP ratios, per-model totals by the exact segmented
fsum kernel.  fp32_full dataset (curves + fitted membound models).

Softmax features are a fixed shape->features map (the reference has none;
SURVEY §8d): elements e = batch*heads*seq^2, flops 5e, int_ops e,
bytes_loaded 4e, bytes_stored 4e, total 8e.
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2603_00549_b200 import load_dataset  # noqa: E402
from paper_2603_00549_b200.aggregate import predict_models  # noqa: E402
from paper_2603_00549_b200.core import (DType, LayerSpec, MatMulShape, MemBoundFeatures,  # noqa: E402
                                        ModelGraph)

HIDDEN = (256, 384, 512, 640, 768, 1024, 1280, 1536, 2048, 2560, 3072, 4096, 5120, 6144)


def block(batch, seq, hidden, mult, heads=None):
    heads = heads or max(1, hidden // 64)
    dh = hidden // heads
    m = batch * seq
    lin = lambda lid, n, k: LayerSpec(lid, "linear", DType.FP32,  # noqa: E731
                                      shape=MatMulShape(batch=1, m=m, n=n, k=k))
    e = float(batch * heads * seq * seq)
    return ModelGraph(f"b{batch}s{seq}h{hidden}x{mult}", (
        lin("attn.q", hidden, hidden), lin("attn.k", hidden, hidden), lin("attn.v", hidden, hidden),
        LayerSpec("attn.scores", "batched_matmul", DType.FP32,
                  shape=MatMulShape(batch=batch * heads, m=seq, n=seq, k=dh)),
        LayerSpec("attn.softmax", "utility:softmax", DType.FP32,
                  features=MemBoundFeatures(flops=5 * e, int_ops=e, bytes_loaded=4 * e,
                                            bytes_stored=4 * e, total_bytes_accessed=8 * e)),
        lin("attn.out", hidden, hidden), lin("mlp.up", mult * hidden, hidden),
        lin("mlp.down", hidden, mult * hidden)), batch_size=batch)


TEMPLATE_IDS = ("attn.q", "attn.k", "attn.v", "attn.scores", "attn.softmax", "attn.out",
                "mlp.up", "mlp.down")


def grid_arrays(params):
    """Vectorised shapes [n, 8, 4] and features [n, 8, 5] of the blocks."""
    import numpy as np
    p = np.array(params, np.int64)           # (batch, seq, hidden, mult)
    b, s, h, r = p.T
    heads = np.maximum(1, h // 64)
    m = b * s
    n = len(p)
    shapes = np.zeros((n, 8, 4), np.int64)
    feats = np.zeros((n, 8, 5), np.float64)
    one = np.ones(n, np.int64)
    for l, (nn, kk) in zip((0, 1, 2, 5, 6, 7), ((h, h), (h, h), (h, h), (h, h), (r * h, h), (h, r * h))):
        shapes[:, l] = np.stack([one, m, nn, kk], 1)
    shapes[:, 3] = np.stack([b * heads, s, s, h // heads], 1)
    e = (b * heads * s * s).astype(np.float64)
    feats[:, 4] = np.stack([5 * e, e, 4 * e, 4 * e, 8 * e], 1)
    return shapes, feats


def main():
    import numpy as np
    from paper_2603_00549_b200.aggregate import TemplateLayer, predict_model_grid
    ds = load_dataset(os.path.join(ROOT, "tests", "golden", "datasets", "fp32_full.json"))
    params = [(b, s, h, r) for b in (1, 2, 4, 8, 16, 32, 64, 128, 256)
              for s in (64, 128, 256, 512, 1024, 2048, 4096, 8192) if b * s < 65536
              for h in HIDDEN for r in (2, 4, 8)]
    fams = ("linear", "linear", "linear", "batched_matmul", "utility:softmax", "linear", "linear", "linear")
    template = [TemplateLayer(i, f, DType.FP32) for i, f in zip(TEMPLATE_IDS, fams)]
    # object API on every 10th model (reference-shaped), as the exactness check
    graphs = [block(*q) for q in params[::10]]
    res = predict_models(graphs, ds)
    for rep in range(3):
        t0 = time.perf_counter()
        shapes, feats = grid_arrays(params)
        lat, tot = predict_model_grid(template, shapes, feats, ds)
        t = time.perf_counter() - t0
    for g_i, r in zip(range(0, len(params), 10), res):
        assert tot[g_i].hex() == r.total_latency_us.hex()
        assert [x.hex() for x in lat[g_i]] == [lp.prediction.latency_us.hex() for lp in r.per_layer]
    best = int(np.argmin(tot))
    print({"C4 models": len(params), "layers": 8 * len(params), "s": t,
           "models_per_s": len(params) / t, "layer_preds_per_s": 8 * len(params) / t,
           "fastest": params[best], "fastest_total_us": float(tot[best]),
           "exact_vs_predict_models": f"{len(res)} models bit-identical (per layer and total)"})


if __name__ == "__main__":
    main()
