"""Device-resident table sets: every (family, dtype,
transpose) triple of a dataset staged in HBM once, for mixed sweeps.

The reference rebuilds PreparedGrid.tables() per grid
(pm2lat/nascache.py:140-241) from the dataset it loaded
(pm2lat/ingest.py:432-445).  A NAS precompute that sweeps many grids of the
same triples re-stages identical tables each time.  DeviceTableSet builds
each triple's flat tables once (host, exactly build_triple_tables), uploads
them on first use, and binds PreparedGrids to the staged handle.  The
dataset fingerprint (pm2lat/ingest.py:130-134) guards reuse: a set built
from one dataset refuses another (StaleCache, as CacheStore.verify does).
"""

from __future__ import annotations

from typing import Dict, Optional, Tuple

from .compute import WaveModel
from .core import DType, TransposeMode
from .errors import StaleCache, ValidationError
from .ingest import Dataset, load_dataset
from .nascache import GridSpec, PreparedGrid
from .tables import build_triple_tables

Triple = Tuple[str, DType, TransposeMode]


class DeviceTableSet:
    def __init__(self, dataset: Dataset, wm: Optional[WaveModel] = None, device: int = 0):
        self.dataset = dataset
        self.wm = wm or WaveModel(sm_count=dataset.device.sm_count)
        self.device = device
        self.fingerprint = dataset.fingerprint()
        self._host: Dict[Triple, tuple] = {}
        for r in dataset.config_map:
            t = (r.family, r.dtype, r.transpose_mode)
            if t not in self._host:
                self._host[t] = build_triple_tables(dataset.config_map, dataset.curves, *t, self.wm)
        self._dev: Dict[Triple, object] = {}

    @classmethod
    def from_json(cls, path, wm: Optional[WaveModel] = None, device: int = 0) -> "DeviceTableSet":
        return cls(load_dataset(path), wm, device)

    def triples(self):
        return sorted(self._host, key=lambda t: (t[0], t[1].value, t[2].value))

    def host_tables(self, family: str, dtype: DType, transpose: TransposeMode) -> dict:
        """The reference's flat arrays of one triple (PreparedGrid.tables())."""
        try:
            return self._host[(family, dtype, transpose)][4]
        except KeyError:
            raise ValidationError(f"dataset has no records for {family}/{dtype.value}/"
                                  f"{transpose.value}") from None

    def tables(self, family: str, dtype: DType, transpose: TransposeMode):
        """The triple's HBM-resident tables (staged on first use)."""
        t = (family, dtype, transpose)
        if t not in self._dev:
            from ._native import DeviceTables
            self._dev[t] = DeviceTables(self.host_tables(*t), self.device)
        return self._dev[t]

    def stage_all(self) -> int:
        """Upload every triple now; returns the number of triples staged."""
        for t in self.triples():
            self.tables(*t)
        return len(self._dev)

    def verify(self, dataset: Dataset) -> None:
        if dataset.fingerprint() != self.fingerprint:
            raise StaleCache("device table set was staged from a different dataset")

    def prepared(self, grid: GridSpec, dataset: Optional[Dataset] = None) -> PreparedGrid:
        """A PreparedGrid for ``grid`` bound to the staged tables of its
        triple (no new upload)."""
        if dataset is not None:
            self.verify(dataset)
        prep = PreparedGrid(self.dataset, grid, self.wm)
        t = (grid.family, grid.dtype, grid.transpose_mode)
        if t in self._host:
            prep._device = self.tables(*t)
        return prep
