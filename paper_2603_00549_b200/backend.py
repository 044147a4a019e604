"""Batch-prediction backend: the plug-in point of the hot path.

Same entry points as pm2lat/backend.py:37-88 — ``predict_grid(prep, jobs,
force_python)``, ``active_backend()``, ``compiled_available()`` — but the
single backend is the sm_100a library (libpm2l_b200.so).  There is no
CPU fallback: a missing library or GPU raises ``BackendUnavailable``, and
``force_python=True`` (which selects the reference's Python loop) is
refused rather than silently ignored.

Extras for device-resident pipelines: ``predict_grid_device`` returns torch
CUDA tensors (optionally with per-point curve id / blocks / waves) and
``predict_grid_all_curves`` evaluates every candidate kernel per shape.
"""

from __future__ import annotations

import numpy as np

from . import _device, _native
from .errors import BackendUnavailable, ValidationError


def active_backend() -> str:
    return "cuda"


def compiled_available() -> bool:
    """True when the sm_100a library is built and a CUDA device is visible."""
    try:
        return _native.device_count() > 0
    except OSError:
        return False


def _axes(prep):
    axes = prep.axis_arrays()
    return [(a.ctypes.data, len(a)) for a in axes], axes


def predict_grid_device(prep, b_lo: int = 0, b_hi=None, verify: bool = False,
                        out=None, stream=None, device: int = 0):
    """Launch the grid kernel for batch indices [b_lo, b_hi) on the device.

    Returns the latency tensor (float64, canonical order) — or, with
    ``verify``, a tuple (latency, curve i32, blocks i64, waves i64).
    Asynchronous on ``stream`` (default: torch's current stream)."""
    dev = _device.device(device)
    nb = len(prep.grid.axes["batch"])
    b_hi = nb if b_hi is None else b_hi
    if not 0 <= b_lo <= b_hi <= nb:
        raise ValidationError(f"batch slice [{b_lo}, {b_hi}) out of range")
    inner = len(prep.grid.axes["m"]) * len(prep.grid.axes["n"]) * len(prep.grid.axes["k"])
    count = (b_hi - b_lo) * inner
    lat = out if out is not None else _device.empty(count, "float64", dev)
    if lat.numel() < count:
        raise ValidationError("output buffer too small")
    curve = blocks = waves = None
    if verify:
        curve = _device.empty(count, "int32", dev)
        blocks = _device.empty(count, "int64", dev)
        waves = _device.empty(count, "int64", dev)
    dt = prep.device_tables(device)
    ptrs, keep = _axes(prep)   # keep the host axis arrays alive across the call
    (pb, lb), (pm, lm), (pn, ln), (pk, lk) = ptrs
    s = _native.stream_handle(stream)
    _native.check(_native.load().pm2l_grid_predict(
        dt.handle, pb, lb, pm, lm, pn, ln, pk, lk, b_lo, b_hi, _native.ptr(lat),
        _native.ptr(curve), _native.ptr(blocks), _native.ptr(waves), s), "pm2l_grid_predict")
    return (lat, curve, blocks, waves) if verify else lat


def predict_grid(prep, jobs: int = 1, force_python: bool = False) -> np.ndarray:
    """Latency (us) of every grid point in canonical (batch, m, n, k) nested
    ascending order; NaN marks unresolved points (backend.py:49-55).

    ``jobs`` is accepted for signature compatibility; the device result is
    independent of it (as the reference guarantees for its thread count)."""
    if force_python:
        raise BackendUnavailable("force_python: the B200 build has no Python/CPU fallback; "
                                 "the reference oracle lives in oracle/ (test-only)")
    card = prep.grid.cardinality
    out = np.empty(card, dtype=np.float64)   # pageable, as backend.py:61 allocates it
    if card == 0:
        return out
    _device.device()
    dt = prep.device_tables(0)
    ptrs, keep = _axes(prep)   # keep the host axis arrays alive across the call
    (pb, lb), (pm, lm), (pn, ln), (pk, lk) = ptrs
    # device kernel into HBM, then the chunked D2H through the library's
    # pinned staging ring + host copy pool straight into ``out``
    _native.check(_native.load().pm2l_grid_predict_host(
        dt.handle, pb, lb, pm, lm, pn, ln, pk, lk, 0, lb, out.ctypes.data),
        "pm2l_grid_predict_host")
    return out


def predict_grid_all_curves(prep, b_lo: int = 0, b_hi=None, stream=None, device: int = 0):
    """Mode X: every (shape, candidate kernel) pair — predict_generic for each
    curve of the grid's triple (compute.py:150-193).  Returns a CUDA float64
    tensor [n_curves, slice cardinality] (NaN for kernels without a curve)."""
    dev = _device.device(device)
    nb = len(prep.grid.axes["batch"])
    b_hi = nb if b_hi is None else b_hi
    inner = len(prep.grid.axes["m"]) * len(prep.grid.axes["n"]) * len(prep.grid.axes["k"])
    count = (b_hi - b_lo) * inner
    C = len(prep.curve_list)
    out = _device.empty((C, count), "float64", dev)
    dt = prep.device_tables(device)
    ptrs, keep = _axes(prep)   # keep the host axis arrays alive across the call
    (pb, lb), (pm, lm), (pn, ln), (pk, lk) = ptrs
    _native.check(_native.load().pm2l_grid_predict_all_curves(
        dt.handle, pb, lb, pm, lm, pn, ln, pk, lk, b_lo, b_hi, _native.ptr(out),
        _native.stream_handle(stream)), "pm2l_grid_predict_all_curves")
    return out


def synchronize():
    """Wait for the device work queued on the current stream."""
    _device.torch().cuda.current_stream().synchronize()


def first_nan(lat) -> int:
    """Flat index of the first NaN of a CUDA float64 tensor (pm2l_nan_scan),
    -1 if none."""
    t = _device.torch()
    first = t.full((1,), -1, dtype=t.int64, device=lat.device)
    _native.check(_native.load().pm2l_nan_scan(lat.data_ptr(), int(lat.numel()), first.data_ptr(),
                                              _native.stream_handle()), "pm2l_nan_scan")
    v = int(first.item())
    return -1 if v < 0 else v
