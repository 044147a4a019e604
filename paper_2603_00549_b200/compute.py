"""Compute-kernel latency prediction — the per-op API of pm2lat/compute.py.

    latency = ref_dur * (v / ref_v) * (ref_thr / thr(v)) * (waves / ref_waves)

Every latency (and every interpolated throughput) is computed on the GPU by
libpm2l_b200.so (``points_curve_kernel``); resolution (exact match, else the
nearest recorded shape by Chebyshev distance in log2 space, ties to the first
record in (m, n, k, batch) order) runs in ``points_kernel``.  The Python layer
validates arguments exactly like the reference (same exceptions, same
messages' meaning) and assembles ``Prediction`` objects.

``WaveModel``, ``block_count`` and ``wave_count`` are the integer tile/wave
model as host utilities for callers that build fixtures or inspect a shape;
the device kernels carry their own u64 implementation of the same formulas
(kernels.cu: blocks_of / ceil_div) and never call these.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import Dict, List, Optional, Tuple

import numpy as np

from .core import (MATMUL_FAMILIES, ROWBLOCK_FAMILIES, VARYING_DIM_NAME, DType, KernelKey,
                   MatMulShape, Prediction, ThroughputCurve, TransposeMode, is_utility_family)
from .errors import (CurveMismatch, InvalidTile, NoConfigAvailable, UnknownFamily,
                     ValidationError)

CLAMP_BELOW = "below_range"
CLAMP_ABOVE = "above_range"
MATCH_EXACT = "exact"
MATCH_NEAREST = "nearest"


@dataclass(frozen=True)
class WaveModel:
    """Blocks per wave = SM count x resident blocks per SM (compute.py:54-75)."""
    sm_count: int
    blocks_per_sm: int = 1

    def __post_init__(self):
        if self.sm_count < 1 or self.blocks_per_sm < 1:
            raise InvalidTile(f"wave model needs sm_count and blocks_per_sm >= 1, got "
                              f"{self.sm_count}/{self.blocks_per_sm}")

    @property
    def blocks_per_wave(self) -> int:
        return self.sm_count * self.blocks_per_sm

    def for_curve(self, curve: ThroughputCurve) -> "WaveModel":
        bps = curve.blocks_per_sm
        return self if bps is None or bps == self.blocks_per_sm else WaveModel(self.sm_count, bps)


def block_count(family: str, shape: MatMulShape, key: KernelKey) -> int:
    """Thread blocks of one launch (compute.py:78-99): GEMM families tile the
    output (partial tiles cost a block; split-K multiplies), row-block
    families launch ceil(batch * k / tile_m) blocks."""
    if family in MATMUL_FAMILIES:
        if key.tile_m < 1 or key.tile_n < 1:
            raise InvalidTile(f"kernel for {family} has tile {key.tile_m}x{key.tile_n}")
        return shape.batch * -(-shape.m // key.tile_m) * -(-shape.n // key.tile_n) * key.split_k
    if family in ROWBLOCK_FAMILIES:
        if key.tile_m < 1:
            raise InvalidTile(f"kernel for {family} has block size {key.tile_m}")
        return -(-(shape.batch * shape.k) // key.tile_m)
    if is_utility_family(family):
        raise UnknownFamily(f"{family} is not a compute family")
    raise UnknownFamily(f"no block model for family {family!r}")


def wave_count(shape: MatMulShape, key: KernelKey, wm: WaveModel) -> int:
    return -(-block_count(key.family, shape, key) // wm.blocks_per_wave)


# ------------------------------------------------------- device curve sets
class _CurveSet:
    """Staged single-triple tables holding explicit curves (no records), for
    predict_generic / interpolate_throughput.  Cached per (curves, wm)."""

    _cache: Dict[tuple, "_CurveSet"] = {}

    def __init__(self, curves: Tuple[ThroughputCurve, ...], wm: WaveModel):
        from .tables import curve_set_tables
        from ._native import DeviceTables
        self.curves = curves
        self.index = {c: i for i, c in enumerate(curves)}
        self.dev = DeviceTables(curve_set_tables(list(curves), wm), 0)

    @classmethod
    def get(cls, curves: Tuple[ThroughputCurve, ...], wm: WaveModel) -> "_CurveSet":
        key = (curves, wm)
        cs = cls._cache.get(key)
        if cs is None:
            if len(cls._cache) > 256:
                cls._cache.clear()
            cs = cls._cache[key] = cls(curves, wm)
        return cs


def _check_pair(key: KernelKey, curve: ThroughputCurve) -> None:
    if curve.kernel != key:
        raise CurveMismatch(f"curve belongs to {curve.kernel.family} algo="
                            f"{curve.kernel.algorithm_id}, not {key.family} "
                            f"algo={key.algorithm_id}")
    expected = VARYING_DIM_NAME[key.family]
    if curve.varying_dim_name != expected:
        raise CurveMismatch(f"curve varies {curve.varying_dim_name!r} but family "
                            f"{key.family} varies {expected!r}")
    if key.family in MATMUL_FAMILIES and (key.tile_m < 1 or key.tile_n < 1):
        raise InvalidTile(f"kernel for {key.family} has tile {key.tile_m}x{key.tile_n}")
    if key.family in ROWBLOCK_FAMILIES and key.tile_m < 1:
        raise InvalidTile(f"kernel for {key.family} has block size {key.tile_m}")


def _shapes_u32(shapes) -> np.ndarray:
    """Shapes as the 16-byte explicit descriptor {b, m, n, k} (u32 each)."""
    a = np.asarray(shapes, dtype=object if _has_big(shapes) else np.int64).reshape(-1, 4)
    if a.size and (a.min() < 1 or a.max() >= (1 << 32)):
        raise ValidationError("shape coordinates must be in [1, 2^32) (the explicit "
                              "descriptor holds u32 coordinates)")
    return np.ascontiguousarray(a.astype(np.uint32))


def _has_big(shapes) -> bool:
    try:
        np.asarray(shapes, dtype=np.int64)
        return False
    except OverflowError:
        return True


_LUT_N = None


def _log2_extension(s: np.ndarray, dev):
    """(coords, log2) device arrays for the query coordinates beyond the
    per-device libm log2 table: math.log2 of each distinct m, n, k >= 2^22
    (the reference resolver's own log2, compute.py:261)."""
    from . import _device, _native
    global _LUT_N
    if _LUT_N is None:
        _LUT_N = int(_native.load().pm2l_points_log2_table_size())
    cols = s[:, 1:]
    big = np.unique(cols[cols >= _LUT_N]) if s.size else np.empty(0, np.uint32)
    if big.size == 0:
        return None, None, 0
    logs = np.array([math.log2(int(v)) for v in big], np.float64)
    return (_device.to_device(np.ascontiguousarray(big, np.uint32), dev),
            _device.to_device(logs, dev), int(big.size))


def predict_curve_batch(shapes, curves: List[ThroughputCurve], curve_ids, wm: WaveModel,
                        detail: bool = False):
    """Device batch of predict_generic over explicit (shape, curve) pairs.

    Returns (latency f64[n], waves u64[n], detail f64[n, 4] or None) with
    detail = (base_us, new_throughput_gflops, wave_scale, waves).  A block
    count past 2^64 (which the reference's unbounded Python integers would
    still carry) raises ValidationError."""
    from . import _device, _native
    dev = _device.device()
    cs = _CurveSet.get(tuple(curves), wm)
    s = _shapes_u32(shapes)
    n = s.shape[0]
    d_s = _device.to_device(s, dev)
    cid = np.ascontiguousarray(curve_ids, dtype=np.int32)
    d_c = _device.to_device(cid, dev)
    lat = _device.empty(n, "float64", dev)
    waves = _device.empty(n, "int32", dev)
    det = _device.empty((n, 4), "float64", dev)
    _native.check(_native.load().pm2l_points_predict_curve(
        cs.dev.handle, _native.ptr(d_s), _native.ptr(d_c), n, _native.ptr(lat),
        _native.ptr(waves), _native.ptr(det), _device.stream()), "pm2l_points_predict_curve")
    lat, det = _device.to_numpy(lat), _device.to_numpy(det)
    bad = np.isnan(lat) & np.array([curves[c] is not None for c in cid], bool)
    if bad.any():
        i = int(np.nonzero(bad)[0][0])
        raise ValidationError(f"shape {tuple(int(x) for x in s[i])}: block count exceeds 2^64")
    w = np.nan_to_num(det[:, 3]).astype(np.uint64)
    return lat, w, det if detail else None


def _interpolate_detail(curve: ThroughputCurve, new_dim: int) -> Tuple[float, Optional[str]]:
    dims = curve.dim_values()
    wm = WaveModel(1)
    _, _, det = predict_curve_batch([(1, 1, 1, new_dim)], [curve], [0], wm, detail=True)
    clamp = CLAMP_BELOW if new_dim < dims[0] else CLAMP_ABOVE if new_dim > dims[-1] else None
    return float(det[0, 1]), clamp


def interpolate_throughput(curve: ThroughputCurve, new_dim: int) -> float:
    """Piecewise-linear throughput at ``new_dim`` (exact at samples, clamped
    outside) — computed by the device (kernels.cu interp_thr)."""
    return _interpolate_detail(curve, new_dim)[0]


def _predict(shape: MatMulShape, key: KernelKey, curve: ThroughputCurve,
             wm: WaveModel) -> Prediction:
    _check_pair(key, curve)
    wm_eff = wm.for_curve(curve)
    lat, waves, det = predict_curve_batch([shape.as_tuple()], [curve], [0], wm, detail=True)
    dims = curve.dim_values()
    clamp = CLAMP_BELOW if shape.k < dims[0] else CLAMP_ABOVE if shape.k > dims[-1] else None
    return Prediction(
        latency_us=float(lat[0]), kernel=key,
        components={"base_us": float(det[0, 0]), "ref_duration_us": curve.ref_duration_us,
                    "varying_value": shape.k, "ref_dim_value": curve.ref_dim_value,
                    "new_throughput_gflops": float(det[0, 1]),
                    "ref_throughput_gflops": curve.ref_throughput, "waves": int(waves[0]),
                    "ref_waves": curve.ref_waves, "wave_scale": float(det[0, 2]),
                    "blocks_per_wave": wm_eff.blocks_per_wave, "clamp": clamp})


def predict_compute(shape: MatMulShape, key: KernelKey, curve: ThroughputCurve,
                    wm: WaveModel) -> Prediction:
    """GEMM families only (compute.py:141-147)."""
    if key.family not in MATMUL_FAMILIES:
        raise UnknownFamily(f"predict_compute handles GEMM families only, got {key.family!r}")
    return _predict(shape, key, curve, wm)


def predict_generic(shape: MatMulShape, key: KernelKey, curve: ThroughputCurve,
                    wm: WaveModel) -> Prediction:
    """Any compute family (compute.py:150-160)."""
    if key.family not in MATMUL_FAMILIES and key.family not in ROWBLOCK_FAMILIES:
        raise UnknownFamily(f"no compute predictor for family {key.family!r}")
    return _predict(shape, key, curve, wm)


def with_component(pred: Prediction, name: str, value) -> Prediction:
    return replace(pred, components={**pred.components, name: value})


# ------------------------------------------------------------- resolution
@dataclass(frozen=True)
class ResolvedConfig:
    key: KernelKey
    match: str
    distance: float


class ConfigResolver:
    """Replays recorded configuration choices (compute.py:211-268).

    Construction validates the config map on the host (an ambiguous map —
    one query recorded with two kernels — raises ValidationError).
    ``resolve`` / ``resolve_batch`` run on the GPU: exact match first, else
    the nearest record by Chebyshev distance in (log2 m, log2 n, log2 k),
    ties to the smaller (m, n, k, batch)."""

    def __init__(self, records, dataset=None, wm: Optional[WaveModel] = None):
        self._records = tuple(records)
        self._dataset = dataset
        self._wm = wm
        self._exact: Dict[tuple, KernelKey] = {}
        self._triples: Dict[tuple, int] = {}
        for r in self._records:
            q = (r.family, r.dtype, r.transpose_mode, r.shape.as_tuple())
            prev = self._exact.get(q)
            if prev is not None and prev != r.chosen_key:
                raise ValidationError(
                    f"ambiguous config map: shape {r.shape.as_tuple()} of ({r.family}, "
                    f"{r.dtype.value}, {r.transpose_mode.value}) recorded with two "
                    f"different kernels")
            self._exact[q] = r.chosen_key
            t = (r.family, r.dtype, r.transpose_mode)
            self._triples[t] = self._triples.get(t, 0) + 1
        self._staged: Dict[tuple, tuple] = {}

    def __len__(self) -> int:
        return len(self._exact)

    def triple_tables(self, family: str, dtype: DType, transpose: TransposeMode):
        """(records in scan order, curve list, rec->curve, key->curve, DeviceTables)."""
        t = (family, dtype, transpose)
        st = self._staged.get(t)
        if st is None:
            from .tables import build_triple_tables
            from ._native import DeviceTables
            curves = self._dataset.curves if self._dataset is not None else {}
            wm = self._wm or WaveModel(self._dataset.device.sm_count if self._dataset else 1)
            recs, clist, rec_curve, index, tables = build_triple_tables(
                self._records, curves, family, dtype, transpose, wm)
            st = self._staged[t] = (recs, clist, rec_curve, index, DeviceTables(tables, 0))
        return st

    def resolve_batch(self, family: str, dtype: DType, transpose: TransposeMode, shapes):
        """Device batch resolution: (record index i32[n], match i8[n],
        distance f64[n]) against this triple's records in scan order."""
        from . import _device, _native
        if not self._triples.get((family, dtype, transpose)):
            raise NoConfigAvailable(f"no recorded configuration for ({family}, {dtype.value}, "
                                    f"{transpose.value})")
        recs, _, _, _, dt = self.triple_tables(family, dtype, transpose)
        s = _shapes_u32(shapes)
        n = s.shape[0]
        dev = _device.device()
        d_s = _device.to_device(s, dev)
        ext_c, ext_l, n_ext = _log2_extension(s, dev)
        lat = _device.empty(n, "float64", dev)
        rec = _device.empty(n, "int32", dev)
        match = _device.empty(n, "int8", dev)
        dist = _device.empty(n, "float64", dev)
        _native.check(_native.load().pm2l_points_predict_ext(
            dt.handle, _native.ptr(d_s), n, _native.ptr(ext_c), _native.ptr(ext_l), n_ext,
            _native.ptr(lat), 0, 0, _native.ptr(match), _native.ptr(rec), _native.ptr(dist), 0,
            _device.stream()), "pm2l_points_predict_ext")
        match = _device.to_numpy(match)
        if (match == -2).any():
            i = int(np.nonzero(match == -2)[0][0])
            raise ValidationError(f"shape {tuple(int(x) for x in s[i])}: invalid coordinate")
        return _device.to_numpy(rec), match, _device.to_numpy(dist)

    def resolve(self, family: str, dtype: DType, transpose_mode: TransposeMode,
                shape: MatMulShape) -> ResolvedConfig:
        exact = self._exact.get((family, dtype, transpose_mode, shape.as_tuple()))
        if exact is not None:   # dictionary hit: no arithmetic involved
            return ResolvedConfig(key=exact, match=MATCH_EXACT, distance=0.0)
        rec, match, dist = self.resolve_batch(family, dtype, transpose_mode,
                                              [shape.as_tuple()])
        recs = self._staged[(family, dtype, transpose_mode)][0]
        return ResolvedConfig(key=recs[int(rec[0])].chosen_key,
                              match=MATCH_EXACT if match[0] == 0 else MATCH_NEAREST,
                              distance=float(dist[0]))


def resolve_config(family: str, dtype: DType, transpose_mode: TransposeMode,
                   shape: MatMulShape, resolver: ConfigResolver) -> KernelKey:
    return resolver.resolve(family, dtype, transpose_mode, shape).key
