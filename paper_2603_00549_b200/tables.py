"""Host-side staging of the reference's flat prediction tables.

``build_triple_tables`` is PreparedGrid.__init__ + PreparedGrid.tables()
(pm2lat/nascache.py:140-241) for one (family, dtype, transpose) triple:
the candidate records in the resolver's scan order, the de-duplicated curve
list, and the flat SoA arrays the device planner (csrc/tables.cpp) consumes.
It performs no prediction arithmetic.
"""

from __future__ import annotations

import math
from typing import Dict, List, Optional

import numpy as np

from .core import MATMUL_FAMILIES, DType, KernelKey, ThroughputCurve, TransposeMode

#: the reference's packed exact-key limit (nascache.py:55-57); the device path
#: does not need it, it only decides whether ``exact_keys`` can be packed.
FAST_COORD_LIMIT = 1 << 16


def build_triple_tables(config_map, curves: Dict[KernelKey, ThroughputCurve], family: str,
                        dtype: DType, transpose: TransposeMode, wm):
    """(records in scan order, curve list, per-record curve index, tables dict)
    for one (family, dtype, transpose) triple — nascache.py:140-241."""
    triple = (family, dtype, transpose)
    records = [r for r in config_map
               if (r.family, r.dtype, r.transpose_mode) == triple]
    records.sort(key=lambda r: (r.shape.m, r.shape.n, r.shape.k, r.shape.batch))
    curve_list: List[Optional[ThroughputCurve]] = []
    index: Dict[KernelKey, int] = {}
    rec_curve: List[int] = []
    for r in records:
        ci = index.get(r.chosen_key)
        if ci is None:
            ci = index[r.chosen_key] = len(curve_list)
            curve_list.append(curves.get(r.chosen_key))
        rec_curve.append(ci if curve_list[ci] is not None else -1)

    n_rec, n_cur = len(records), len(curve_list)
    coords = np.array([r.shape.as_tuple() for r in records], dtype=np.uint64).reshape(n_rec, 4)
    # libm log2 — the value the canonical scalar resolver uses (compute.py:239,261)
    log_m = np.array([math.log2(r.shape.m) for r in records], dtype=np.float64)
    log_n = np.array([math.log2(r.shape.n) for r in records], dtype=np.float64)
    log_k = np.array([math.log2(r.shape.k) for r in records], dtype=np.float64)
    cand = np.array(rec_curve, dtype=np.int64)
    tables = {"log_m": log_m, "log_n": log_n, "log_k": log_k, "cand_curve": cand,
              "exact_coords": np.ascontiguousarray(coords), "exact_coords_curve": cand.copy()}
    if n_rec == 0 or int(coords.max()) < FAST_COORD_LIMIT:
        packed = ((coords[:, 0] << np.uint64(48)) | (coords[:, 1] << np.uint64(32))
                  | (coords[:, 2] << np.uint64(16)) | coords[:, 3]) if n_rec else \
            np.zeros(0, np.uint64)
        order = np.argsort(packed, kind="stable")
        tables["exact_keys"] = packed[order]
        tables["exact_curve"] = cand[order]
    else:
        tables["exact_keys"] = None
        tables["exact_curve"] = None
    tables.update(curve_arrays(curve_list, wm))
    return records, curve_list, rec_curve, index, tables


def curve_arrays(curve_list: List[Optional[ThroughputCurve]], wm) -> dict:
    """Per-curve SoA arrays (nascache.py:196-226); a None entry (recorded
    kernel without a throughput curve) gets no samples."""
    n_cur = len(curve_list)
    offsets = np.zeros(n_cur + 1, dtype=np.int64)
    dims: List[float] = []
    thrs: List[float] = []
    out = {n: np.zeros(n_cur, np.float64) for n in ("ref_dim", "ref_dur", "ref_thr", "ref_waves")}
    out.update({n: np.zeros(n_cur, np.uint64) for n in ("tile_m", "tile_n", "split_k",
                                                          "blocks_per_wave")})
    rowblock = np.zeros(n_cur, np.uint8)
    for ci, c in enumerate(curve_list):
        if c is not None:
            dims.extend(float(s.dim_value) for s in c.samples)
            thrs.extend(s.throughput_gflops for s in c.samples)
            out["ref_dim"][ci] = float(c.ref_dim_value)
            out["ref_dur"][ci] = c.ref_duration_us
            out["ref_thr"][ci] = c.ref_throughput
            out["ref_waves"][ci] = float(c.ref_waves)
            out["tile_m"][ci] = c.kernel.tile_m
            out["tile_n"][ci] = c.kernel.tile_n
            out["split_k"][ci] = c.kernel.split_k
            out["blocks_per_wave"][ci] = wm.for_curve(c).blocks_per_wave
            rowblock[ci] = 0 if c.kernel.family in MATMUL_FAMILIES else 1
        offsets[ci + 1] = len(dims)
    out.update(sample_offsets=offsets, sample_dims=np.array(dims, np.float64),
               sample_thrs=np.array(thrs, np.float64), family_rowblock=rowblock)
    return out


def curve_set_tables(curve_list: List[ThroughputCurve], wm) -> dict:
    """Tables of explicit curves with zero candidate records (predict_generic)."""
    t = curve_arrays(curve_list, wm)
    t.update(log_m=np.zeros(0), log_n=np.zeros(0), log_k=np.zeros(0),
             cand_curve=np.zeros(0, np.int64), exact_coords=np.zeros((0, 4), np.uint64),
             exact_coords_curve=np.zeros(0, np.int64), exact_keys=np.zeros(0, np.uint64),
             exact_curve=np.zeros(0, np.int64))
    return t
