"""TEST INFRASTRUCTURE — the CPU oracle.  Not part of the product.

Only tests/, __graft_entry__.smoke() and bench.py (its cpu_baseline leg and
``--impl reference``) may import this package, and only as the checker /
the reference arm — never as the thing measured or shipped.

* ``liboracle.so`` (built from pm2l_oracle.c by ``make``): plain-C
  restatement of the reference path, each function citing the reference
  file:line it follows.  Pinned against tests/golden/ (reference outputs).
* ``_ref/_kernels*.so`` (``make ref``, only where /root/reference exists):
  the reference's own Cython kernel compiled from its source, used as the
  ``kind: "reference"`` CPU baseline.  The GPU box gets the prebuilt file.
"""

from __future__ import annotations

import ctypes as C
import importlib.util
import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
REF_DIR = os.path.join(HERE, "_ref")

_lib = None


def build(ref: bool = True) -> None:
    """Compile liboracle.so (and the reference Cython kernel when
    /root/reference is present)."""
    subprocess.run(["make", "-s", "liboracle.so"], cwd=HERE, check=True)
    if ref and os.path.exists("/root/reference/pkg/src/pm2lat/_kernels.pyx"):
        subprocess.run(["make", "-s", "ref", f"PY={sys.executable}"], cwd=HERE, check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build(ref=False)
        L = C.CDLL(LIB)
        p, i64 = C.c_void_p, C.c_int64
        L.pm2lo_grid.argtypes = [p, p, i64, p, i64, p, i64, p, i64, i64, i64, p, p, p, p]
        L.pm2lo_points.argtypes = [p, p, i64, p, p, p, p, p, p]
        L.pm2lo_points_curve.argtypes = [p, p, p, i64, p, p, p]
        L.pm2lo_membound.argtypes = [p, p, i64, p, p, p, i64, p, p]
        L.pm2lo_fsum.argtypes = [p, i64]
        L.pm2lo_fsum.restype = C.c_double
        L.pm2lo_segment_fsum.argtypes = [p, p, i64, p]
        L.pm2lo_grid_error.argtypes = [p, p, i64, i64, p, p, p, p, p]
        L.pm2lo_partition.argtypes = [p, p, i64, p, p, p, p]
        L.pm2lo_partition.restype = i64
        _lib = L
    return _lib


# --------------------------------------------------------------- tables view
class _View(C.Structure):
    _fields_ = [
        ("n_records", C.c_int64), ("exact_keys", C.c_void_p), ("exact_coords", C.c_void_p),
        ("exact_curve", C.c_void_p), ("log_m", C.c_void_p), ("log_n", C.c_void_p),
        ("log_k", C.c_void_p), ("cand_curve", C.c_void_p), ("n_curves", C.c_int64),
        ("sample_offsets", C.c_void_p), ("sample_dims", C.c_void_p),
        ("sample_thrs", C.c_void_p), ("ref_dim", C.c_void_p), ("ref_dur", C.c_void_p),
        ("ref_thr", C.c_void_p), ("ref_waves", C.c_void_p), ("tile_m", C.c_void_p),
        ("tile_n", C.c_void_p), ("split_k", C.c_void_p), ("blocks_per_wave", C.c_void_p),
        ("family_rowblock", C.c_void_p)]


def _view(tables: dict, use_coords: bool):
    keep = []

    def arr(name, dt):
        a = tables.get(name)
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a.ctypes.data

    v = _View()
    v.n_records = len(tables["cand_curve"])
    if use_coords or tables.get("exact_keys") is None:
        v.exact_coords = arr("exact_coords", np.uint64)
        v.exact_curve = arr("exact_coords_curve", np.int64)
    else:
        v.exact_keys = arr("exact_keys", np.uint64)
        v.exact_curve = arr("exact_curve", np.int64)
    for n in ("log_m", "log_n", "log_k", "sample_dims", "sample_thrs", "ref_dim", "ref_dur",
              "ref_thr", "ref_waves"):
        setattr(v, n, arr(n, np.float64))
    v.cand_curve = arr("cand_curve", np.int64)
    v.n_curves = len(tables["sample_offsets"]) - 1
    v.sample_offsets = arr("sample_offsets", np.int64)
    for n in ("tile_m", "tile_n", "split_k", "blocks_per_wave"):
        setattr(v, n, arr(n, np.uint64))
    v.family_rowblock = arr("family_rowblock", np.uint8)
    return v, keep


def grid(tables: dict, axes, b_lo=0, b_hi=None, verify=True, use_coords=False):
    """Oracle latencies (and curve/blocks/waves) of a canonical grid slice."""
    B, M, N, K = (np.ascontiguousarray(a, dtype=np.uint64) for a in axes)
    b_hi = len(B) if b_hi is None else b_hi
    n = (b_hi - b_lo) * len(M) * len(N) * len(K)
    out = np.empty(n, np.float64)
    cur = np.empty(n, np.int32) if verify else None
    blk = np.empty(n, np.uint64) if verify else None
    wav = np.empty(n, np.uint64) if verify else None
    v, keep = _view(tables, use_coords)
    P = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    lib().pm2lo_grid(C.byref(v), B.ctypes.data, len(B), M.ctypes.data, len(M), N.ctypes.data,
                     len(N), K.ctypes.data, len(K), b_lo, b_hi, out.ctypes.data, P(cur),
                     P(blk), P(wav))
    return (out, cur, blk, wav) if verify else out


def points(tables: dict, shapes):
    s = np.ascontiguousarray(shapes, dtype=np.uint32).reshape(-1, 4)
    n = s.shape[0]
    lat = np.empty(n, np.float64)
    cur = np.empty(n, np.int32)
    wav = np.empty(n, np.uint32)
    mat = np.empty(n, np.int8)
    rec = np.empty(n, np.int32)
    dist = np.empty(n, np.float64)
    v, keep = _view(tables, True)
    lib().pm2lo_points(C.byref(v), s.ctypes.data, n, lat.ctypes.data, cur.ctypes.data,
                       wav.ctypes.data, mat.ctypes.data, rec.ctypes.data, dist.ctypes.data)
    return lat, cur, wav, mat, rec, dist


def points_curve(tables: dict, shapes, curves):
    s = np.ascontiguousarray(shapes, dtype=np.uint32).reshape(-1, 4)
    c = np.ascontiguousarray(curves, dtype=np.int32)
    n = s.shape[0]
    lat = np.empty(n, np.float64)
    wav = np.empty(n, np.uint32)
    det = np.empty((n, 4), np.float64)
    v, keep = _view(tables, True)
    lib().pm2lo_points_curve(C.byref(v), s.ctypes.data, c.ctypes.data, n, lat.ctypes.data,
                             wav.ctypes.data, det.ctypes.data)
    return lat, wav, det


def membound(features, model_ids, weights, intercepts, floors):
    f = np.ascontiguousarray(features, np.float64).reshape(-1, 5)
    m = np.ascontiguousarray(model_ids, np.int32)
    w = np.ascontiguousarray(weights, np.float64).reshape(-1, 5)
    b = np.ascontiguousarray(intercepts, np.float64)
    fl = np.ascontiguousarray(floors, np.float64)
    n = f.shape[0]
    out = np.empty(n, np.float64)
    flo = np.empty(n, np.uint8)
    lib().pm2lo_membound(f.ctypes.data, m.ctypes.data, n, w.ctypes.data, b.ctypes.data,
                         fl.ctypes.data, len(b), out.ctypes.data, flo.ctypes.data)
    return out, flo.astype(bool)


def segment_fsum(values, offsets):
    v = np.ascontiguousarray(values, np.float64)
    o = np.ascontiguousarray(offsets, np.int64)
    out = np.empty(len(o) - 1, np.float64)
    lib().pm2lo_segment_fsum(v.ctypes.data, o.ctypes.data, len(o) - 1, out.ctypes.data)
    return out


def grid_error(dims, thrs, stride, truth=None, scan_off=None, rational=None):
    """curvefit.grid_error_report per interval: (max_rel_err f64[n-1], argmax i64[n-1])."""
    d = np.ascontiguousarray(dims, np.int64)
    t = np.ascontiguousarray(thrs, np.float64)
    tr = None if truth is None else np.ascontiguousarray(truth, np.float64)
    so = None if scan_off is None else np.ascontiguousarray(scan_off, np.int64)
    r = None if rational is None else np.ascontiguousarray(rational, np.float64)
    err = np.empty(len(d) - 1, np.float64)
    arg = np.empty(len(d) - 1, np.int64)
    P = lambda a: None if a is None else a.ctypes.data  # noqa: E731
    lib().pm2lo_grid_error(d.ctypes.data, t.ctypes.data, len(d), int(stride), P(tr), P(so), P(r),
                           err.ctypes.data, arg.ctypes.data)
    return err, arg


def partition(lat_a, lat_b, transfer=None):
    """partition_two_device's scan: (stage_a, stage_b, bottleneck, best cut)."""
    la = np.ascontiguousarray(lat_a, np.float64)
    lb = np.ascontiguousarray(lat_b, np.float64)
    tr = None if transfer is None else np.ascontiguousarray(transfer, np.float64)
    n = len(la)
    sa, sb, bn = (np.empty(n + 1, np.float64) for _ in range(3))
    best = lib().pm2lo_partition(la.ctypes.data, lb.ctypes.data, n,
                                 None if tr is None else tr.ctypes.data, sa.ctypes.data,
                                 sb.ctypes.data, bn.ctypes.data)
    return sa, sb, bn, int(best)


# ------------------------------------------------- the reference's own kernel
def reference_kernels():
    """The reference Cython module compiled into _ref/ (or None)."""
    for name in os.listdir(REF_DIR) if os.path.isdir(REF_DIR) else ():
        if name.startswith("_kernels") and name.endswith(".so"):
            spec = importlib.util.spec_from_file_location("_kernels", os.path.join(REF_DIR, name))
            mod = importlib.util.module_from_spec(spec)
            spec.loader.exec_module(mod)
            return mod
    return None


def reference_predict_grid_tiles(kernels, tables: dict, axes, threads: int) -> np.ndarray:
    """The reference's Cython predict_grid_slice (unmodified) over every host
    thread: the grid is cut into (batch value, m range) sub-grids, each one
    contiguous in the canonical output, and each computed by one nogil call
    (_kernels.pyx:76-133) from a thread pool.  Per-point arithmetic does not
    depend on the other axis values, so the output equals the single call's."""
    B, M, N, K = (np.ascontiguousarray(a, dtype=np.uint64) for a in axes)
    nN, nK = len(N), len(K)
    inner = len(M) * nN * nK
    out = np.empty(len(B) * inner, np.float64)
    t = tables
    per_b = max(1, -(-threads // max(1, len(B))))
    m_bounds = np.linspace(0, len(M), min(per_b, max(1, len(M))) + 1, dtype=int)
    tasks = [(b, int(m0), int(m1)) for b in range(len(B))
             for m0, m1 in zip(m_bounds[:-1], m_bounds[1:]) if m1 > m0]

    def run(task):
        b, m0, m1 = task
        Ms = np.ascontiguousarray(M[m0:m1])
        o = b * inner + m0 * nN * nK
        kernels.predict_grid_slice(
            B, Ms, N, K, b, b + 1, t["exact_keys"], t["exact_curve"], t["log_m"], t["log_n"],
            t["log_k"], t["cand_curve"], t["sample_offsets"], t["sample_dims"],
            t["sample_thrs"], t["ref_dim"], t["ref_dur"], t["ref_thr"], t["ref_waves"],
            t["tile_m"], t["tile_n"], t["split_k"], t["blocks_per_wave"],
            t["family_rowblock"], out[o:o + (m1 - m0) * nN * nK])

    with ThreadPoolExecutor(max_workers=max(1, threads)) as pool:
        for f in [pool.submit(run, task) for task in tasks]:
            f.result()
    return out


def reference_predict_grid(kernels, tables: dict, axes, jobs: int = 1) -> np.ndarray:
    """The reference's _predict_grid_compiled (backend.py:58-88): thread pool
    over batch slabs, each calling the Cython predict_grid_slice (nogil)."""
    B, M, N, K = (np.ascontiguousarray(a, dtype=np.uint64) for a in axes)
    inner = len(M) * len(N) * len(K)
    out = np.empty(len(B) * inner, np.float64)
    t = tables

    def run(lo, hi):
        kernels.predict_grid_slice(
            B, M, N, K, lo, hi, t["exact_keys"], t["exact_curve"], t["log_m"], t["log_n"],
            t["log_k"], t["cand_curve"], t["sample_offsets"], t["sample_dims"],
            t["sample_thrs"], t["ref_dim"], t["ref_dur"], t["ref_thr"], t["ref_waves"],
            t["tile_m"], t["tile_n"], t["split_k"], t["blocks_per_wave"],
            t["family_rowblock"], out[lo * inner:hi * inner])

    jobs = max(1, min(jobs, len(B)))
    if jobs == 1:
        run(0, len(B))
    else:
        bounds = np.linspace(0, len(B), jobs + 1, dtype=int)
        with ThreadPoolExecutor(max_workers=jobs) as pool:
            for f in [pool.submit(run, int(lo), int(hi))
                      for lo, hi in zip(bounds[:-1], bounds[1:]) if hi > lo]:
                f.result()
    return out
