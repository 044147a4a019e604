"""ctypes binding of libpm2l_b200.so (include/pm2l.h).

The library is loaded from the package directory (built in-tree by
``_build.build()``).  There is no CPU fallback: if the library is missing or
no CUDA device is visible, every compute entry point raises
``BackendUnavailable`` instead of silently computing elsewhere.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import BackendUnavailable, DeviceError, ValidationError

# PM2L_LIB_PATH: diagnostic builds only (tools/row_timing.py)
_LIB_PATH = os.environ.get("PM2L_LIB_PATH") or os.path.join(
    os.path.dirname(os.path.abspath(__file__)), "libpm2l_b200.so")

PM2L_OK, PM2L_ERR_INVALID, PM2L_ERR_CUDA, PM2L_ERR_NOMEM, PM2L_ERR_NODEVICE = 0, -1, -2, -3, -4

_p = C.c_void_p
_i64 = C.c_int64
_i32 = C.c_int


class TablesView(C.Structure):
    """Mirror of pm2l_tables_view."""
    _fields_ = [
        ("n_records", _i64), ("exact_keys", _p), ("exact_coords", _p), ("exact_curve", _p),
        ("log_m", _p), ("log_n", _p), ("log_k", _p), ("cand_curve", _p),
        ("n_curves", _i64), ("sample_offsets", _p), ("sample_dims", _p), ("sample_thrs", _p),
        ("ref_dim", _p), ("ref_dur", _p), ("ref_thr", _p), ("ref_waves", _p),
        ("tile_m", _p), ("tile_n", _p), ("split_k", _p), ("blocks_per_wave", _p),
        ("family_rowblock", _p),
    ]


#: every symbol include/pm2l.h declares, with (restype, argtypes)
SIGNATURES = {
    "pm2l_abi_version": (_i32, []),
    "pm2l_source_hash": (C.c_char_p, []),
    "pm2l_last_error": (C.c_char_p, []),
    "pm2l_device_count": (_i32, []),
    "pm2l_tables_create": (_i32, [C.POINTER(TablesView), _i32, C.POINTER(_p)]),
    "pm2l_tables_destroy": (_i32, [_p]),
    "pm2l_tables_groups": (_i64, [_p]),
    "pm2l_grid_predict": (_i32, [_p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _i64,
                                 _p, _p, _p, _p, _p]),
    "pm2l_grid_plan_create": (_i32, [_p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _i64,
                                     C.POINTER(_p)]),
    "pm2l_grid_plan_launch": (_i32, [_p, _p, _p, _p, _p, _p, _i32, _p]),
    "pm2l_grid_plan_info": (_i32, [_p, C.POINTER(_i64)]),
    "pm2l_grid_plan_kernel": (_i32, [_p, _p, _i32]),
    "pm2l_grid_plan_destroy": (_i32, [_p]),
    "pm2l_grid_dplan_create": (_i32, [_p, _i64, _i64, _i64, _i64, C.POINTER(_p)]),
    "pm2l_grid_dplan_launch": (_i32, [_p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _i64,
                                      _p, _p, _p, _p, _p, _i32, _p]),
    "pm2l_grid_dplan_status": (_i32, [_p, C.POINTER(C.c_uint32)]),
    "pm2l_grid_dplan_kernel": (_i32, [_p]),
    "pm2l_grid_dplan_fixups": (_i32, [_p, C.POINTER(_i64)]),
    "pm2l_grid_dplan_destroy": (_i32, [_p]),
    "pm2l_nan_scan": (_i32, [_p, _i64, _p, _p]),
    "pm2l_grid_predict_host": (_i32, [_p, _p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _i64,
                                      _p]),
    "pm2l_grid_predict_all_curves": (_i32, [_p, _p, _i64, _p, _i64, _p, _i64, _p, _i64,
                                            _i64, _i64, _p, _p]),
    "pm2l_points_predict": (_i32, [_p, _p, _i64, _p, _p, _p, _p, _p, _p, _p]),
    "pm2l_points_predict_ext": (_i32, [_p, _p, _i64, _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p,
                                       _p]),
    "pm2l_points_log2_table_size": (_i64, []),
    "pm2l_points_predict_curve": (_i32, [_p, _p, _p, _i64, _p, _p, _p, _p]),
    "pm2l_membound_predict": (_i32, [_p, _p, _i64, _p, _p, _p, _i64, _p, _p, _p]),
    "pm2l_membound_predict_raw": (_i32, [_p, _p, _i64, _p, _p, _p, _i64, _p, _p, _p, _p]),
    "pm2l_segment_fsum": (_i32, [_p, _p, _i64, _p, _p]),
    "pm2l_grid_error_report": (_i32, [_p, _p, _i64, _i64, _p, _p, _p, _p, _p, _p]),
    "pm2l_partition_scan": (_i32, [_p, _p, _i64, _p, _p, _p, _p, _p, _p]),
    "pm2l_store_encode_workspace": (_i64, [_i64]),
    "pm2l_store_encode": (_i32, [_p, _i64, _p, _p, _i64, _p, _i64, _p, _i64, _p, _p, _p, _p]),
    "pm2l_store_lookup": (_i32, [_p, _i64, _p, _p, _p, _i64, _p, _p, _p]),
    "pm2l_predict_grid_slice": (_i32, [_p, _i64, _p, _i64, _p, _i64, _p, _i64, _i64, _i64,
                                       _p, _p, _i64, _p, _p, _p, _p, _p, _p, _p, _i64,
                                       _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
}

_lib = None
_lock = threading.Lock()


def library_path() -> str:
    return _LIB_PATH


def load(required: bool = True):
    """The loaded CDLL (or None when missing and not required)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB_PATH):
                if not required:
                    return None
                raise BackendUnavailable(
                    f"{_LIB_PATH} is not built (run __graft_entry__.build() or "
                    f"python -m paper_2603_00549_b200._build); there is no CPU fallback")
            lib = C.CDLL(_LIB_PATH)
            ab = bool(os.environ.get("PM2L_LIB_PATH"))  # diagnostic / A-B builds
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(lib, name, None)
                if fn is None and ab:   # an older build: entry points it lacks stay unbound
                    continue
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            from . import _build
            try:
                want = _build.source_hash()
            except OSError:      # sources not shipped: nothing to compare against
                want = None
            if os.environ.get("PM2L_LIB_PATH"):  # diagnostic / A-B builds
                want = None
            got = lib.pm2l_source_hash().decode()
            if want is not None and got != want:
                raise BackendUnavailable(
                    f"{_LIB_PATH} was built from different sources ({got} != {want}); "
                    f"rebuild with __graft_entry__.build()")
            _lib = lib
    return _lib


def device_count() -> int:
    lib = load(required=False)
    return 0 if lib is None else int(lib.pm2l_device_count())


def check(rc: int, what: str) -> None:
    if rc == PM2L_OK:
        return
    msg = load().pm2l_last_error().decode("utf-8", "replace")
    if rc == PM2L_ERR_NODEVICE:
        raise BackendUnavailable(f"{what}: {msg}")
    if rc == PM2L_ERR_INVALID:
        raise ValidationError(f"{what}: {msg}")
    raise DeviceError(f"{what}: {msg} (status {rc})")


def require_gpu():
    """Load the library and make sure a CUDA device is visible."""
    lib = load()
    if lib.pm2l_device_count() < 1:
        raise BackendUnavailable("no CUDA device visible: the B200 build has no CPU fallback")
    return lib


def ptr(a) -> int:
    """Address of a numpy array / torch tensor (0 for None)."""
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return a.ctypes.data
    return int(a.data_ptr())


_RAW_STREAM = None


def stream_handle(stream=None) -> int:
    """cudaStream_t of ``stream`` or of torch's current stream on the current
    device (the raw binding: no Stream object per call)."""
    global _RAW_STREAM
    import torch
    if stream is not None:
        return int(stream.cuda_stream)
    if _RAW_STREAM is None:
        _RAW_STREAM = getattr(torch._C, "_cuda_getCurrentRawStream", False)
    if _RAW_STREAM:
        return int(_RAW_STREAM(torch.cuda.current_device()))
    return int(torch.cuda.current_stream().cuda_stream)


class DeviceTables:
    """Owning wrapper of a pm2l_tables handle (HBM-resident staged tables)."""

    def __init__(self, tables: dict, device: int = 0):
        lib = require_gpu()
        keep = {}

        def arr(name, dtype):
            a = tables.get(name)
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dtype)
            keep[name] = a
            return a.ctypes.data

        view = TablesView()
        view.n_records = len(tables["cand_curve"])
        view.exact_keys = arr("exact_keys", np.uint64) if tables.get("exact_coords") is None else None
        view.exact_coords = arr("exact_coords", np.uint64)
        view.exact_curve = arr("exact_curve" if tables.get("exact_coords") is None
                               else "exact_coords_curve", np.int64)
        for name in ("log_m", "log_n", "log_k"):
            setattr(view, name, arr(name, np.float64))
        view.cand_curve = arr("cand_curve", np.int64)
        view.n_curves = len(tables["sample_offsets"]) - 1
        view.sample_offsets = arr("sample_offsets", np.int64)
        view.sample_dims = arr("sample_dims", np.float64)
        view.sample_thrs = arr("sample_thrs", np.float64)
        for name in ("ref_dim", "ref_dur", "ref_thr", "ref_waves"):
            setattr(view, name, arr(name, np.float64))
        for name in ("tile_m", "tile_n", "split_k", "blocks_per_wave"):
            setattr(view, name, arr(name, np.uint64))
        view.family_rowblock = arr("family_rowblock", np.uint8)
        handle = C.c_void_p()
        check(lib.pm2l_tables_create(C.byref(view), device, C.byref(handle)), "pm2l_tables_create")
        self._lib = lib
        self.handle = handle
        self.device = device
        self.n_curves = int(view.n_curves)
        self.n_records = int(view.n_records)

    @property
    def groups(self) -> int:
        return int(self._lib.pm2l_tables_groups(self.handle))

    def close(self):
        if self.handle:
            self._lib.pm2l_tables_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class GridPlan:
    """Owning wrapper of pm2l_grid_plan: a grid slice staged once, launched
    many times (kernels only)."""

    def __init__(self, tables: DeviceTables, axes, b_lo: int = 0, b_hi=None):
        lib = require_gpu()
        arrs = [np.ascontiguousarray(a, dtype=np.uint64) for a in axes]
        b_hi = len(arrs[0]) if b_hi is None else b_hi
        handle = C.c_void_p()
        args = []
        for a in arrs:
            args += [a.ctypes.data, len(a)]
        check(lib.pm2l_grid_plan_create(tables.handle, *args, b_lo, b_hi, C.byref(handle)),
              "pm2l_grid_plan_create")
        self._lib = lib
        self._tables = tables  # keep alive
        self.handle = handle
        info = (_i64 * 4)()
        check(lib.pm2l_grid_plan_info(handle, info), "pm2l_grid_plan_info")
        self.cardinality, self.n_fixups, self.workspace_bytes, self.staged_bytes = \
            (int(x) for x in info)

    def launch(self, out_lat, curve=None, blocks=None, waves=None, nan_stats=None,
               stages: int = 7, stream=None):
        check(self._lib.pm2l_grid_plan_launch(
            self.handle, ptr(out_lat), ptr(curve), ptr(blocks), ptr(waves), ptr(nan_stats),
            stages, stream_handle(stream)), "pm2l_grid_plan_launch")

    def kernel_path(self, out_lat, verify: bool = False) -> int:
        """0 sweep, 1 sweep + tie mask, 2 one-class closed form, 3 lookup."""
        rc = self._lib.pm2l_grid_plan_kernel(self.handle, ptr(out_lat), int(verify))
        if rc < 0:
            check(rc, "pm2l_grid_plan_kernel")
        return rc

    def close(self):
        if self.handle:
            self._lib.pm2l_grid_plan_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceGridPlanner:
    """Owning wrapper of pm2l_grid_dplan: per-slice planning on the GPU.
    ``launch`` takes DEVICE axis tensors (canonical GridSpec order) and runs
    the planner kernel + grid kernel in the stream; nothing returns to the
    host between slices (CUDA-graph capturable)."""

    def __init__(self, tables: DeviceTables, max_batch: int, max_m: int, max_n: int, max_k: int):
        lib = require_gpu()
        handle = C.c_void_p()
        check(lib.pm2l_grid_dplan_create(tables.handle, max_batch, max_m, max_n, max_k,
                                         C.byref(handle)), "pm2l_grid_dplan_create")
        self._lib = lib
        self._tables = tables
        self.handle = handle

    def launch(self, axes, out_lat, b_lo: int = 0, b_hi=None, curve=None, blocks=None,
               waves=None, nan_stats=None, stages: int = 7, stream=None):
        B, M, N, K = axes
        b_hi = len(B) if b_hi is None else b_hi
        check(self._lib.pm2l_grid_dplan_launch(
            self.handle, ptr(B), len(B), ptr(M), len(M), ptr(N), len(N), ptr(K), len(K),
            b_lo, b_hi, ptr(out_lat), ptr(curve), ptr(blocks), ptr(waves), ptr(nan_stats),
            stages, stream_handle(stream)), "pm2l_grid_dplan_launch")

    def status(self) -> int:
        """Sticky axis-contract violations since the last call (0: none)."""
        v = C.c_uint32()
        check(self._lib.pm2l_grid_dplan_status(self.handle, C.byref(v)), "pm2l_grid_dplan_status")
        return int(v.value)

    def kernel_path(self) -> int:
        return int(self._lib.pm2l_grid_dplan_kernel(self.handle))

    def fixups(self) -> int:
        n = _i64()
        check(self._lib.pm2l_grid_dplan_fixups(self.handle, C.byref(n)), "pm2l_grid_dplan_fixups")
        return int(n.value)

    def close(self):
        if self.handle:
            self._lib.pm2l_grid_dplan_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
