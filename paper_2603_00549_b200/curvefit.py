"""Interpolation-grid audit on the device.

``grid_error_report`` mirrors pm2lat/curvefit.py:192-219: for every sample
interval of a throughput curve, the worst relative error of the
piecewise-linear interpolation the prediction path uses
(compute.interpolate_throughput) against a truth curve, over every integer
dim of the interval (strided once the span exceeds ``max_points``, the
interval's upper sample always included).  The scan, the interpolation, the
errors and the per-interval first-maximum reductions run in
``grid_error_kernel`` (csrc/audit.cu).  A truth given as a rational trend
(anything with float attributes a, b, c, d and y = (a*x + b)/(c*x + d), as
the reference's PlantedCurve and RationalFit are) is evaluated on the
device; any other callable is evaluated here once per scanned dim (it is
Python code) and its values shipped to the device.

The rational least-squares fit itself (curvefit.fit_rational) is an
off-path diagnostic and is not part of this package.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Tuple

import numpy as np

from .core import ThroughputCurve
from .errors import ValidationError


@dataclass(frozen=True)
class IntervalError:
    lo_dim: int
    hi_dim: int
    max_rel_err: float
    argmax_dim: int


@dataclass(frozen=True)
class GridErrorReport:
    """Worst-case piecewise-linear interpolation error versus a reference
    curve, densely scanned per sample interval."""

    max_rel_err: float
    argmax_dim: int
    intervals: Tuple[IntervalError, ...]

    def to_json_obj(self) -> dict:
        return {
            "max_rel_err": self.max_rel_err,
            "argmax_dim": self.argmax_dim,
            "intervals": [
                {"lo_dim": iv.lo_dim, "hi_dim": iv.hi_dim,
                 "max_rel_err": iv.max_rel_err, "argmax_dim": iv.argmax_dim}
                for iv in self.intervals
            ],
        }


@dataclass(frozen=True)
class RationalTrend:
    """y = (a*x + b) / (c*x + d) (the reference's PlantedCurve / RationalFit
    evaluation, oracle.py:58-59, curvefit.py:37-38)."""

    a: float
    b: float
    c: float
    d: float

    def __call__(self, x) -> float:
        return (self.a * x + self.b) / (self.c * x + self.d)


def _rational(oracle):
    try:
        coef = tuple(getattr(oracle, n) for n in ("a", "b", "c", "d"))
    except AttributeError:
        return None
    if all(isinstance(v, float) for v in coef) and callable(oracle):
        return coef
    return None


def scan_dims(dims, max_points: int = 200_000):
    """(stride, per-interval scan lists) exactly as curvefit.py:199-208."""
    span = dims[-1] - dims[0] + 1
    stride = max(1, span // max_points)
    scans = []
    for lo, hi in zip(dims, dims[1:]):
        scan = list(range(lo, hi, stride))
        if scan[-1] != hi:
            scan.append(hi)
        scans.append(scan)
    return stride, scans


def grid_error_report(curve: ThroughputCurve, oracle: Callable[[int], float],
                      max_points: int = 200_000) -> GridErrorReport:
    """Scan every integer dim in [min sample, cap] (strided once the range
    exceeds ``max_points``, sample endpoints always included) and report
    |interpolated - oracle| / oracle per interval and globally."""
    from . import _device, _native
    dims = list(curve.dim_values())
    if len(dims) < 2:
        raise ValidationError("a throughput curve has at least two samples")
    thrs = np.array([s.throughput_gflops for s in curve.samples], np.float64)
    span = dims[-1] - dims[0] + 1
    stride = max(1, span // max_points)
    dev = _device.device()
    t = _device.torch()
    d_dims = _device.to_device(np.array(dims, np.int64), dev)
    d_thr = _device.to_device(thrs, dev)
    coef = _rational(oracle)
    truth = off = None
    rat = None
    if coef is None:
        _, scans = scan_dims(dims, max_points)
        host = np.array([float(oracle(d)) for scan in scans for d in scan], np.float64)
        offs = np.concatenate([[0], np.cumsum([len(s) for s in scans])[:-1]]).astype(np.int64)
        truth = _device.to_device(host, dev)
        off = _device.to_device(offs, dev)
    else:
        rat = np.array(coef, np.float64)
    n_iv = len(dims) - 1
    err = t.empty(n_iv, dtype=t.float64, device=dev)
    arg = t.empty(n_iv, dtype=t.int64, device=dev)
    _native.check(_native.load().pm2l_grid_error_report(
        _native.ptr(d_dims), _native.ptr(d_thr), len(dims), stride, _native.ptr(truth),
        _native.ptr(off), _native.ptr(rat), _native.ptr(err), _native.ptr(arg),
        _device.stream()), "pm2l_grid_error_report")
    err, arg = err.cpu().numpy(), arg.cpu().numpy()
    intervals = tuple(IntervalError(lo_dim=lo, hi_dim=hi, max_rel_err=float(e), argmax_dim=int(a))
                      for lo, hi, e, a in zip(dims, dims[1:], err, arg))
    worst = (-1.0, dims[0])
    for iv in intervals:          # the reference's strict-> scan over intervals
        if iv.max_rel_err > worst[0]:
            worst = (iv.max_rel_err, iv.argmax_dim)
    return GridErrorReport(max_rel_err=worst[0], argmax_dim=worst[1], intervals=intervals)


__all__ = ["IntervalError", "GridErrorReport", "RationalTrend", "grid_error_report", "scan_dims"]
