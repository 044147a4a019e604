"""Grid precomputation (the NAS latency cache) and its binary lookup store.

Drop-in for pm2lat/nascache.py.  ``GridSpec`` / ``PreparedGrid`` /
``precompute`` / ``CacheStore`` keep the reference's names, semantics and
the byte-exact store format (magic "PM2L", u16 version, u32 header length,
sorted JSON header, then 40-byte big-endian records ``>QQQQd``,
nascache.py:48-53,309-333).  The per-point prediction runs on the GPU
(backend.predict_grid); the tables handed to the device are the reference's
``PreparedGrid.tables()`` arrays (nascache.py:174-241) plus unpacked exact
coordinates so grids with coordinates >= 2^16 stay on the device too.
"""

from __future__ import annotations

import hashlib
import itertools
import json
import math
import mmap
import struct
import time
from dataclasses import dataclass
from typing import Dict, Iterator, List, Optional, Sequence, Tuple

import numpy as np

from .compute import ConfigResolver, WaveModel
from .core import (COMPUTE_FAMILIES, MATMUL_FAMILIES, DType, KernelKey, ThroughputCurve,
                   TransposeMode, check_family)
from .errors import CacheFormatError, MissingEntry, StaleCache, UnresolvedPoint, ValidationError
from .ingest import Dataset
from .tables import FAST_COORD_LIMIT, build_triple_tables

MAGIC = b"PM2L"
FORMAT_VERSION = 1
AXIS_ORDER = ("batch", "m", "n", "k")
_KEY_STRUCT = struct.Struct(">QQQQ")
_REC_STRUCT = struct.Struct(">QQQQd")
RECORD_SIZE = _REC_STRUCT.size
#: waves / blocks must stay exactly representable as doubles (2^53)
EXACT_INT_LIMIT = 1 << 53

_RECORD_DTYPE = np.dtype([("b", ">u8"), ("m", ">u8"), ("n", ">u8"), ("k", ">u8"),
                          ("lat", ">f8")])


@dataclass(frozen=True)
class GridSpec:
    """Per-axis value lists (sorted, unique, >= 1; missing axis = (1,)) for
    one compute family / dtype / transpose (nascache.py:60-127)."""
    family: str
    dtype: DType
    transpose_mode: TransposeMode
    axes: Dict[str, Tuple[int, ...]]

    def __post_init__(self):
        check_family(self.family)
        if self.family not in COMPUTE_FAMILIES:
            raise ValidationError(f"grids cover compute families only, got {self.family!r}")
        unknown = set(self.axes) - set(AXIS_ORDER)
        norm = {}
        for name in AXIS_ORDER:
            vals = tuple(sorted(int(v) for v in self.axes.get(name, (1,))))
            if not vals:
                raise ValidationError(f"axis {name!r} must be non-empty")
            if len(set(vals)) != len(vals):
                raise ValidationError(f"axis {name!r} has duplicate values")
            if vals[0] < 1:
                raise ValidationError(f"axis {name!r} values must be >= 1")
            norm[name] = vals
        if unknown:
            raise ValidationError(f"unknown grid axes {sorted(unknown)}")
        object.__setattr__(self, "axes", norm)

    @property
    def cardinality(self) -> int:
        return math.prod(len(self.axes[a]) for a in AXIS_ORDER)

    def shape(self) -> Tuple[int, int, int, int]:
        return tuple(len(self.axes[a]) for a in AXIS_ORDER)

    def iter_points(self) -> Iterator[Tuple[int, int, int, int]]:
        return itertools.product(*(self.axes[a] for a in AXIS_ORDER))

    def to_json_obj(self) -> dict:
        return {"family": self.family, "dtype": self.dtype.value,
                "transpose_mode": self.transpose_mode.value,
                "axes": {a: list(self.axes[a]) for a in AXIS_ORDER}}

    @classmethod
    def from_json_obj(cls, obj) -> "GridSpec":
        try:
            fam = obj["family"]
            return cls(family=fam, dtype=DType.parse(obj["dtype"]),
                       transpose_mode=TransposeMode.parse(
                           obj.get("transpose_mode", "tn" if fam == "linear" else "nn")),
                       axes={a: tuple(v) for a, v in obj["axes"].items()})
        except KeyError as exc:
            raise ValidationError(f"grid spec missing field {exc.args[0]!r}") from None

    def fingerprint(self) -> str:
        text = json.dumps(self.to_json_obj(), sort_keys=True, separators=(",", ":"))
        return hashlib.sha256(text.encode()).hexdigest()


class PreparedGrid:
    """Everything the device backend needs for one grid (nascache.py:130-245).

    ``tables()`` returns the reference's flat arrays; ``device_tables()``
    stages them in HBM once (cached on this object)."""

    def __init__(self, dataset: Dataset, grid: GridSpec, wm: WaveModel):
        self.grid = grid
        self.wm = wm
        self.dataset = dataset
        self.resolver = ConfigResolver(dataset.config_map, dataset=dataset, wm=wm)
        (self.records, self.curve_list, self.record_curve_idx, self._curve_index,
         self._tables) = build_triple_tables(dataset.config_map, dataset.curves, grid.family,
                                             grid.dtype, grid.transpose_mode, wm)
        coords = [v for r in self.records for v in r.shape.as_tuple()]
        max_coord = max(coords + [grid.axes[a][-1] for a in AXIS_ORDER])
        #: the reference's Cython eligibility flag, kept for API parity; the
        #: device path serves every grid regardless
        self.fast_path_ok = bool(self.records) and max_coord < FAST_COORD_LIMIT
        self._device = None
        self._check_exact_integers()

    def _check_exact_integers(self):
        """Waves go through (double)waves / ref_waves; the reference's Python
        path uses unbounded ints, so the device result is only identical while
        blocks stay below 2^53.  Reject grids that could exceed it."""
        ax = self.grid.axes
        bmax, mmax, nmax, kmax = (ax[a][-1] for a in AXIS_ORDER)
        worst = 0
        for c in self.curve_list:
            if c is None:
                continue
            key = c.kernel
            if key.family in MATMUL_FAMILIES:
                worst = max(worst, bmax * -(-mmax // key.tile_m) * -(-nmax // key.tile_n)
                            * key.split_k)
            else:
                worst = max(worst, bmax * kmax)
        if worst >= EXACT_INT_LIMIT:
            raise ValidationError(
                f"grid block counts reach {worst} >= 2^53: waves would not be exact doubles")

    def has_candidates(self) -> bool:
        return bool(self.records)

    def tables(self) -> dict:
        return self._tables

    def axis_arrays(self) -> Tuple[np.ndarray, ...]:
        return tuple(np.array(self.grid.axes[a], dtype=np.uint64) for a in AXIS_ORDER)

    def device_tables(self, device: int = 0):
        if self._device is None or self._device.device != device:
            from ._native import DeviceTables
            self._device = DeviceTables(self._tables, device)
        return self._device

    def curve_index(self, key: KernelKey) -> int:
        return self._curve_index[key]


@dataclass(frozen=True)
class PrecomputeSummary:
    total_points: int
    entries_written: int
    skipped: int
    elapsed_s: float
    mean_us_per_prediction: float
    backend: str

    def to_json_obj(self) -> dict:
        return {"total_points": self.total_points, "entries_written": self.entries_written,
                "skipped": self.skipped, "elapsed_s": self.elapsed_s,
                "mean_us_per_prediction": self.mean_us_per_prediction,
                "backend": self.backend}


def point_at(grid: GridSpec, flat_index: int) -> Tuple[int, int, int, int]:
    """Coordinates of a flat index in canonical (batch, m, n, k) order."""
    idx = np.unravel_index(int(flat_index), grid.shape())
    return tuple(grid.axes[a][int(i)] for a, i in zip(AXIS_ORDER, idx))


def encode_records(grid: GridSpec, latencies: np.ndarray) -> np.ndarray:
    """Big-endian 40-byte records of every resolved point, canonical order
    (the byte layout of nascache.py:325-333, vectorised)."""
    nb, nm, nn, nk = grid.shape()
    keep = ~np.isnan(latencies)
    flat = np.nonzero(keep)[0]
    ib, im, jn, ik = np.unravel_index(flat, (nb, nm, nn, nk))
    rec = np.empty(flat.size, dtype=_RECORD_DTYPE)
    for name, ax, idx in (("b", "batch", ib), ("m", "m", im), ("n", "n", jn), ("k", "k", ik)):
        rec[name] = np.asarray(grid.axes[ax], dtype=np.uint64)[idx]
    rec["lat"] = latencies[flat]
    return rec


def encode_records_device(grid: GridSpec, latencies, b_lo: int = 0, device: int = 0) -> np.ndarray:
    """encode_records on the B200 (pm2l_store_encode): ``latencies`` is the
    CUDA float64 tensor of batch indices [b_lo, b_lo + len/inner) of the
    grid; records are built, compacted and byte-swapped on the device and
    only the record bytes come back."""
    from . import _device, _native
    t = _device.torch()
    dev = _device.device(device)
    n = int(latencies.numel())
    nb, nm, nn, nk = grid.shape()
    inner = nm * nn * nk
    if n == 0:
        return np.empty(0, _RECORD_DTYPE)
    if n % inner:
        raise ValidationError("latency count is not a whole number of batch planes")
    b_hi = b_lo + n // inner
    if not 0 <= b_lo < b_hi <= nb:
        raise ValidationError(f"batch slice [{b_lo}, {b_hi}) out of range")
    axes = [t.from_numpy(np.ascontiguousarray(np.asarray(grid.axes[a], dtype=np.uint64)))
            .to(dev) for a in AXIS_ORDER]
    axes[0] = axes[0][b_lo:b_hi].contiguous()
    lib = _native.load()
    ws = t.empty(int(lib.pm2l_store_encode_workspace(n)), dtype=t.uint8, device=dev)
    rec = t.empty(n * RECORD_SIZE, dtype=t.uint8, device=dev)
    count = t.zeros(1, dtype=t.int64, device=dev)
    lat = latencies.contiguous()
    _native.check(lib.pm2l_store_encode(
        lat.data_ptr(), n, axes[0].data_ptr(), axes[1].data_ptr(), nm, axes[2].data_ptr(), nn,
        axes[3].data_ptr(), nk, ws.data_ptr(), rec.data_ptr(), count.data_ptr(),
        _native.stream_handle()), "pm2l_store_encode")
    c = int(count.item())
    # pinned landing buffer (torch's caching host allocator: reused across
    # calls), one DMA of the record bytes; the array keeps the buffer alive
    host = t.empty(c * RECORD_SIZE, dtype=t.uint8, pin_memory=True)
    if c:
        host.copy_(rec[:c * RECORD_SIZE])
    return host.numpy().view(_RECORD_DTYPE)


def write_store(path, grid: GridSpec, dataset: Dataset, latencies: np.ndarray = None,
                records: np.ndarray = None) -> int:
    """Write the store (nascache.py:308-333) from host latencies, or from
    records already encoded (encode_records_device)."""
    rec = records if records is not None else encode_records(grid, latencies)
    header = {"device_id": dataset.device.device_id,
              "dataset_fingerprint": dataset.fingerprint(),
              "grid_fingerprint": grid.fingerprint(),
              "entry_count": int(rec.size), "grid": grid.to_json_obj(),
              "coord_order": list(AXIS_ORDER)}
    hb = json.dumps(header, sort_keys=True, separators=(",", ":")).encode("utf-8")
    with open(path, "wb") as fh:
        fh.write(MAGIC)
        fh.write(struct.pack(">H", FORMAT_VERSION))
        fh.write(struct.pack(">I", len(hb)))
        fh.write(hb)
        fh.write(memoryview(np.ascontiguousarray(rec)).cast("B"))
    return int(rec.size)


def precompute(grid: GridSpec, dataset: Dataset, wm: Optional[WaveModel], out_path,
               jobs: int = 1, skip_unresolved: bool = False) -> PrecomputeSummary:
    """Predict every grid point on the GPU and write the store
    (nascache.py:280-342): the timed region covers table preparation and
    prediction, an unresolved point aborts naming the FIRST offending
    coordinates unless ``skip_unresolved``."""
    from . import backend
    wm = wm or WaveModel(sm_count=dataset.device.sm_count)
    prep = PreparedGrid(dataset, grid, wm)
    total = grid.cardinality
    start = time.perf_counter()
    lat = backend.predict_grid_device(prep) if total else None
    if lat is not None:
        backend.synchronize()
    elapsed = time.perf_counter() - start
    # the records are encoded and compacted on the device (pm2l_store_encode)
    rec = encode_records_device(grid, lat) if total else encode_records(grid, np.empty(0))
    skipped = total - int(rec.size)
    if skipped and not skip_unresolved:
        first = backend.first_nan(lat)
        b, m, n, k = point_at(grid, first)
        raise UnresolvedPoint(
            f"grid point batch={b} m={m} n={n} k={k} ({grid.family}, {grid.dtype.value}, "
            f"{grid.transpose_mode.value}) has no usable kernel configuration")
    write_store(out_path, grid, dataset, records=rec)
    return PrecomputeSummary(total_points=total, entries_written=total - skipped,
                             skipped=skipped, elapsed_s=elapsed,
                             mean_us_per_prediction=elapsed / total * 1e6 if total else 0.0,
                             backend=backend.active_backend())


class CacheStore:
    """Read side of the store: memory-mapped binary search over the sorted
    fixed-width records (nascache.py:345-430)."""

    def __init__(self, path):
        self.path = path
        self._mm = None
        self._fh = open(path, "rb")
        try:
            if self._fh.read(4) != MAGIC:
                raise CacheFormatError(f"{path}: bad magic")
            raw = self._fh.read(6)
            if len(raw) < 6:
                raise CacheFormatError(f"{path}: truncated header")
            version, hlen = struct.unpack(">HI", raw)
            if version != FORMAT_VERSION:
                raise CacheFormatError(f"{path}: unsupported format version {version}")
            try:
                self.header = json.loads(self._fh.read(hlen).decode("utf-8"))
            except ValueError:
                raise CacheFormatError(f"{path}: unreadable header") from None
            self._records_at = 10 + hlen
            size = self._fh.seek(0, 2) - self._records_at
            if size < 0 or size % RECORD_SIZE:
                raise CacheFormatError(f"{path}: truncated record section")
            self.entry_count = size // RECORD_SIZE
            if self.entry_count != self.header.get("entry_count"):
                raise CacheFormatError(f"{path}: header claims {self.header.get('entry_count')} "
                                       f"entries, file has {self.entry_count}")
            if self.entry_count:
                self._mm = mmap.mmap(self._fh.fileno(), 0, access=mmap.ACCESS_READ)
        except Exception:
            self._fh.close()
            raise

    def close(self):
        if self._mm is not None:
            self._mm.close()
            self._mm = None
        self._fh.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def __len__(self):
        return self.entry_count

    def verify(self, dataset: Optional[Dataset] = None, grid: Optional[GridSpec] = None) -> None:
        if dataset is not None and dataset.fingerprint() != self.header.get("dataset_fingerprint"):
            raise StaleCache(f"{self.path}: store was built from a different dataset")
        if grid is not None and grid.fingerprint() != self.header.get("grid_fingerprint"):
            raise StaleCache(f"{self.path}: store was built from a different grid")

    def records(self) -> np.ndarray:
        """All records as a structured big-endian array (zero-copy view)."""
        if not self.entry_count:
            return np.zeros(0, _RECORD_DTYPE)
        return np.frombuffer(self._mm, dtype=_RECORD_DTYPE, count=self.entry_count,
                             offset=self._records_at)

    def lookup(self, batch: int, m: int, n: int, k: int) -> float:
        needle = _KEY_STRUCT.pack(batch, m, n, k)
        lo, hi = 0, self.entry_count
        while lo < hi:
            mid = (lo + hi) // 2
            off = self._records_at + mid * RECORD_SIZE
            key = self._mm[off:off + 32]
            if key < needle:
                lo = mid + 1
            elif key > needle:
                hi = mid
            else:
                return struct.unpack(">d", self._mm[off + 32:off + 40])[0]
        raise MissingEntry(f"point batch={batch} m={m} n={n} k={k} is not in the store")

    def device_records(self, device: int = 0):
        """The record section staged in HBM once (a CUDA uint8 tensor)."""
        from . import _device
        cache = self.__dict__.setdefault("_dev_records", {})
        if device not in cache:
            t = _device.torch()
            raw = np.frombuffer(self._mm, np.uint8, count=self.entry_count * RECORD_SIZE,
                                offset=self._records_at) if self.entry_count else np.zeros(8, np.uint8)
            cache[device] = t.from_numpy(raw.copy()).to(_device.device(device))
        return cache[device]

    def lookup_many(self, points, missing: str = "raise", device: int = 0) -> np.ndarray:
        """lookup() for an (n, 4) array of (batch, m, n, k) points at once on
        the B200 (pm2l_store_lookup): a binary search per point over the
        staged records, or a direct index when the store holds every point of
        its grid.  missing="raise" raises MissingEntry naming the first absent
        point (as lookup would); missing="nan" returns NaN for it."""
        from . import _device, _native
        if missing not in ("raise", "nan"):
            raise ValidationError("missing must be 'raise' or 'nan'")
        q = np.ascontiguousarray(np.asarray(points, dtype=np.uint64).reshape(-1, 4))
        n = len(q)
        if n == 0:
            return np.empty(0, np.float64)
        t = _device.torch()
        dev = _device.device(device)
        rec = self.device_records(device)
        qd = t.from_numpy(q).to(dev)
        out = t.empty(n, dtype=t.float64, device=dev)
        first = t.full((1,), -1, dtype=t.int64, device=dev)
        axes_ptr = lens_ptr = None
        keep = []
        grid = self.header.get("grid")
        if grid and self.entry_count:
            axes = [np.ascontiguousarray(np.asarray(grid["axes"][a], dtype=np.uint64)) for a in AXIS_ORDER]
            if int(np.prod([len(a) for a in axes])) == self.entry_count:
                dax = [t.from_numpy(a).to(dev) for a in axes]
                ptrs = np.array([a.data_ptr() for a in dax], np.uint64)
                lens = np.array([len(a) for a in axes], np.int64)
                keep = [dax, ptrs, lens]
                axes_ptr, lens_ptr = ptrs.ctypes.data, lens.ctypes.data
        _native.check(_native.load().pm2l_store_lookup(
            rec.data_ptr(), self.entry_count, axes_ptr, lens_ptr, qd.data_ptr(), n,
            out.data_ptr(), first.data_ptr(), _native.stream_handle()), "pm2l_store_lookup")
        f = int(first.item())
        del keep
        if f >= 0 and missing == "raise":
            b, m, nn, k = (int(v) for v in q[f])
            raise MissingEntry(f"point batch={b} m={m} n={nn} k={k} is not in the store")
        return out.cpu().numpy()

    def iter_entries(self) -> Iterator[Tuple[Tuple[int, int, int, int], float]]:
        for r in self.records():
            yield (int(r["b"]), int(r["m"]), int(r["n"]), int(r["k"])), float(r["lat"])


def lookup(store: CacheStore, point: Sequence[int]) -> float:
    b, m, n, k = (int(v) for v in point)
    return store.lookup(b, m, n, k)
