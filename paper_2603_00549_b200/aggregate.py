"""Whole-model latency: per-layer predictions + exact per-model totals.

Drop-in for ``ModelPredictor`` / ``predict_model`` (pm2lat/aggregate.py:105-196),
plus ``predict_models`` for batches of graphs (the NAS whole-model sweep).
All layer latencies come from the GPU, batched across every layer of every
graph: compute layers are resolved (``points_kernel``) and predicted
(``points_curve_kernel``), utility layers go through ``membound_kernel``,
and the totals are the correctly-rounded sums of each model's layers
(``segment_fsum_kernel``, bit-identical to ``math.fsum``, aggregate.py:193).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .compute import (CLAMP_ABOVE, CLAMP_BELOW, MATCH_EXACT, MATCH_NEAREST, ConfigResolver,
                      WaveModel, _check_pair)
from .core import (COMPUTE_FAMILIES, FAMILY_LINEAR, DType, KernelKey, LayerSpec, ModelGraph,
                   Prediction, TransposeMode, is_utility_family, utility_kernel_name)
from .errors import (InsufficientData, NoConfigAvailable, PredictionError, UnresolvedLayer,
                     ValidationError)
from .ingest import Dataset
from .membound import DEFAULT_LAUNCH_FLOOR_US, MemBoundModel, fit

_NP_OF: Dict[object, np.dtype] = {}


def _np_dtype(tdtype):
    """numpy dtype of a torch dtype (cached)."""
    d = _NP_OF.get(tdtype)
    if d is None:
        import torch
        d = _NP_OF[tdtype] = torch.empty(0, dtype=tdtype).numpy().dtype
    return d

PREDICTOR_COMPUTE = "compute"
PREDICTOR_MEMBOUND = "membound"
DEFAULT_TRANSPOSE = {FAMILY_LINEAR: TransposeMode.TN}


def default_transpose(family: str) -> TransposeMode:
    return DEFAULT_TRANSPOSE.get(family, TransposeMode.NN)


@dataclass(frozen=True)
class LayerPrediction:
    layer_id: str
    prediction: Prediction
    predictor_kind: str


@dataclass(frozen=True)
class ModelPrediction:
    model_name: str
    total_latency_us: float
    per_layer: Tuple[LayerPrediction, ...]
    flags: Tuple[Tuple[str, str], ...]

    def to_json_obj(self) -> dict:
        return {"model_name": self.model_name, "total_latency_us": self.total_latency_us,
                "per_layer": [{"layer_id": lp.layer_id, "latency_us": lp.prediction.latency_us,
                               "predictor_kind": lp.predictor_kind,
                               "components": dict(lp.prediction.components)}
                              for lp in self.per_layer],
                "flags": [{"layer_id": lid, "flag": f} for lid, f in self.flags]}


class ModelPredictor:
    """Dataset + lookup structures (resolver, fitted membound models)."""

    def __init__(self, dataset: Dataset, wm: Optional[WaveModel] = None,
                 membound_floor_us: float = DEFAULT_LAUNCH_FLOOR_US):
        self.dataset = dataset
        self.wm = wm or WaveModel(sm_count=dataset.device.sm_count)
        self.floor_us = membound_floor_us
        self.resolver = ConfigResolver(dataset.config_map, dataset=dataset, wm=self.wm)
        self._membound: Dict[Tuple[str, DType], MemBoundModel] = {
            (m.kernel_name, m.dtype): m for m in dataset.membound_models}
        self._curves = None

    def membound_model(self, kernel_name: str, dtype: DType) -> MemBoundModel:
        got = self._membound.get((kernel_name, dtype))
        if got is not None:
            return got
        recs = [(r.features, r.latency_us) for r in self.dataset.membound_records
                if r.kernel_name == kernel_name and r.dtype == dtype]
        if not recs:
            raise UnresolvedLayer(f"no fitted model or records for utility kernel "
                                  f"{kernel_name!r} ({dtype.value})")
        try:
            model = fit(recs, kernel_name, dtype, train_device_id=self.dataset.device.device_id)
        except InsufficientData as exc:
            raise UnresolvedLayer(str(exc)) from None
        self._membound[(kernel_name, dtype)] = model
        return model

    def all_curves(self):
        if self._curves is None:
            self._curves = list(self.dataset.curves.values())
            self._curve_pos = {c.kernel: i for i, c in enumerate(self._curves)}
        return self._curves

    def predict_layers(self, layers: Sequence[LayerSpec]):
        """Device batch over layers: [(Prediction, kind, flags)] in order.
        Raises like the reference on the first unresolvable layer."""
        return self._predict_layers(layers)[0]

    def _predict_layers(self, layers: Sequence[LayerSpec], offsets=None):
        """predict_layers, plus (with segment ``offsets`` over ``layers``) the
        correctly rounded per-segment totals, computed on the device inside
        the same pipeline.  Returns (out, totals or None).

        One host->device copy per input kind, then every kernel back to back
        on the stream (resolution per triple, record -> curve map, explicit-
        curve prediction, membound with and without the floor) and ONE
        device->host copy of every output."""
        from . import _device, _native
        from .compute import _log2_extension, _shapes_u32
        n = len(layers)
        out: List[Optional[tuple]] = [None] * n
        errors: Dict[int, Exception] = {}   # the reference raises at the FIRST bad layer

        def wrap(i, exc):
            if isinstance(exc, UnresolvedLayer):
                return exc
            return type(exc)(f"layer {layers[i].layer_id!r}: {exc}")

        by_triple: Dict[tuple, List[int]] = {}
        util_idx: List[int] = []
        for i, layer in enumerate(layers):
            if is_utility_family(layer.family):
                if layer.features is None:
                    errors[i] = UnresolvedLayer(f"utility layer {layer.layer_id!r} carries no "
                                                f"features")
                else:
                    util_idx.append(i)
            elif layer.family not in COMPUTE_FAMILIES:
                errors[i] = UnresolvedLayer(f"layer {layer.layer_id!r}: no predictor for family "
                                            f"{layer.family!r}")
            elif layer.shape is None:
                errors[i] = UnresolvedLayer(f"compute layer {layer.layer_id!r} carries no shape")
            else:
                tr = layer.transpose_mode or default_transpose(layer.family)
                by_triple.setdefault((layer.family, layer.dtype, tr), []).append(i)
        for triple, idx in list(by_triple.items()):
            if not self.resolver._triples.get(triple):
                exc = NoConfigAvailable(f"no recorded configuration for ({triple[0]}, "
                                        f"{triple[1].value}, {triple[2].value})")
                for i in idx:
                    errors[i] = wrap(i, exc)
                del by_triple[triple]
        # utility layers: fitted (or on-demand refit) membound models
        models: List[MemBoundModel] = []
        pos: Dict[tuple, int] = {}
        util_ok, mids = [], []
        for i in util_idx:
            name = utility_kernel_name(layers[i].family)
            mk = (name, layers[i].dtype)
            try:
                if mk not in pos:
                    models.append(self.membound_model(name, layers[i].dtype))
                    pos[mk] = len(models) - 1
            except PredictionError as exc:
                errors[i] = wrap(i, exc)
                continue
            util_ok.append(i)
            mids.append(pos[mk])

        compute_idx = [i for idx in by_triple.values() for i in idx]
        nc, nu = len(compute_idx), len(util_ok)
        dev = _device.device()
        t = _device.torch()
        lib = _native.load()
        sh = None
        if nc:
            try:
                sh = _shapes_u32([layers[i].shape.as_tuple() for i in compute_idx])
            except PredictionError as exc:
                for i in compute_idx:
                    errors[i] = wrap(i, exc)
                nc = 0
        # ---- device pipeline: two host->device copies (one integer blob,
        # one float blob, through pinned staging), every kernel back to back
        # on the stream, one device->host copy of every output
        nseg = 0 if offsets is None else len(offsets) - 1
        ints = np.concatenate([
            sh.astype(np.int64).ravel() if nc else np.zeros(0, np.int64),
            np.asarray(mids, np.int64), np.asarray(compute_idx[:nc], np.int64),
            np.asarray(util_ok, np.int64),
            np.zeros(0, np.int64) if offsets is None else np.asarray(offsets, np.int64)])
        floats = np.zeros(0, np.float64)
        if nu:
            floats = np.concatenate([
                np.array([layers[i].features.as_vector() for i in util_ok], np.float64).ravel(),
                np.array([m.weights for m in models], np.float64).ravel(),
                np.array([m.intercept for m in models], np.float64),
                np.full(len(models), self.floor_us), np.full(len(models), -np.inf)])
        s = _device.stream()
        d_int = _staged_upload(ints, dev)
        d_flt = _staged_upload(floats, dev) if nu else None
        o = 4 * nc
        d_mid = d_int[o:o + nu]
        o += nu
        d_posc = d_int[o:o + nc]
        o += nc
        d_posu = d_int[o:o + nu]
        o += nu
        d_off = d_int[o:o + nseg + 1] if offsets is not None else None
        # every output in ONE device buffer (f64 slots; the int32 / int8
        # outputs live in their own slots), copied back once
        lay_n = n if offsets is not None else 0
        tot_n = nseg if offsets is not None else 0
        sizes = [nc, nc, nc, 4 * nc, nc, nu, nu, nu, lay_n, tot_n]   # rec|cur, match, dist, det, lat, mlat, raw, flo, lay, tot
        starts = [0]
        for z in sizes:
            starts.append(starts[-1] + int(z))
        buf = t.empty(int(starts[-1]), dtype=t.float64, device=dev)
        bp = buf.data_ptr()
        sl = lambda k: buf[starts[k]:starts[k + 1]]  # noqa: E731
        if nc:
            d_sh = d_int[:4 * nc].to(t.int32)   # u32 descriptors (int32 bits)
            ext_c, ext_l, n_ext = _log2_extension(sh, dev)
            o = 0
            for triple, idx in by_triple.items():
                dt = self.resolver.triple_tables(*triple)[4]
                k = len(idx)
                # rec (int32) and curve (int32) share slot 0; match (int8) slot 1
                _native.check(lib.pm2l_points_predict_ext(
                    dt.handle, d_sh.data_ptr() + 16 * o, k, _native.ptr(ext_c), _native.ptr(ext_l),
                    n_ext, bp + 8 * (starts[4] + o), bp + 8 * starts[0] + 4 * o, 0,
                    bp + 8 * starts[1] + o, bp + 8 * starts[0] + 4 * (nc + o),
                    bp + 8 * (starts[2] + o), bp + 8 * (starts[3] + 4 * o), s),
                    "pm2l_points_predict_ext")
                o += k
            if offsets is not None:
                sl(8)[d_posc] = sl(4)
        if nu:
            nf, nw, nm = 5 * nu, 5 * len(models), len(models)
            ids = d_mid.to(t.int32)
            base = d_flt.data_ptr()
            _native.check(lib.pm2l_membound_predict_raw(
                base, ids.data_ptr(), nu, base + 8 * nf, base + 8 * (nf + nw),
                base + 8 * (nf + nw + nm), nm, bp + 8 * starts[5], bp + 8 * starts[7],
                bp + 8 * starts[6], s), "pm2l_membound_predict_raw")
            if offsets is not None:
                sl(8)[d_posu] = sl(5)
        totals = None
        if offsets is not None and nseg > 0:
            _native.check(lib.pm2l_segment_fsum(bp + 8 * starts[8], d_off.data_ptr(), nseg,
                                                bp + 8 * starts[9], s), "pm2l_segment_fsum")
        host = _staged_download(buf)
        v = lambda k, dt_: host[8 * starts[k]:8 * starts[k + 1]].view(dt_)  # noqa: E731
        if offsets is not None and nseg > 0:
            totals = v(9, np.float64).copy()
        if nc:
            ints32 = v(0, np.int32)
            cur, rec = ints32[:nc], ints32[nc:2 * nc]
            match = v(1, np.int8)[:nc]
            dist = v(2, np.float64)
            det = v(3, np.float64).reshape(nc, 4)
            lat = v(4, np.float64)
        if nu:
            mlat, raw, flo = v(5, np.float64), v(6, np.float64), v(7, np.uint8)[:nu]
        if nc:
            o = 0
            for triple, idx in by_triple.items():
                recs, clist = self.resolver.triple_tables(*triple)[:2]
                for j, i in enumerate(idx, start=o):
                    if match[j] == -2:
                        errors[i] = wrap(i, ValidationError(
                            f"shape {layers[i].shape.as_tuple()}: invalid coordinate"))
                        continue
                    key = recs[int(rec[j])].chosen_key
                    if match[j] == -3:
                        errors[i] = wrap(i, ValidationError(
                            f"shape {layers[i].shape.as_tuple()}: block count exceeds 2^64"))
                        continue
                    if cur[j] < 0:
                        errors[i] = UnresolvedLayer(
                            f"layer {layers[i].layer_id!r}: resolved kernel has no throughput "
                            f"curve (family={layers[i].family}, algo={key.algorithm_id})")
                        continue
                    c = clist[int(cur[j])]
                    try:
                        _check_pair(key, c)
                    except PredictionError as exc:
                        errors[i] = wrap(i, exc)
                        continue
                    m = MATCH_EXACT if match[j] == 0 else MATCH_NEAREST
                    kk = layers[i].shape.k
                    dims = c.dim_values()
                    clamp = CLAMP_BELOW if kk < dims[0] else CLAMP_ABOVE if kk > dims[-1] else None
                    comps = {"base_us": float(det[j, 0]), "ref_duration_us": c.ref_duration_us,
                             "varying_value": kk, "ref_dim_value": c.ref_dim_value,
                             "new_throughput_gflops": float(det[j, 1]),
                             "ref_throughput_gflops": c.ref_throughput, "waves": int(det[j, 3]),
                             "ref_waves": c.ref_waves, "wave_scale": float(det[j, 2]),
                             "blocks_per_wave": self.wm.for_curve(c).blocks_per_wave,
                             "clamp": clamp, "config_match": m}
                    flags = (["nearest_config"] if m == MATCH_NEAREST else []) + \
                        ([clamp] if clamp else [])
                    out[i] = (Prediction(float(lat[j]), key, comps), PREDICTOR_COMPUTE, flags)
                o += len(idx)
        if nu:
            for j, i in enumerate(util_ok):
                key = KernelKey.for_utility(models[mids[j]].kernel_name, layers[i].dtype)
                comps = {"raw_us": float(raw[j]), "floor_us": self.floor_us,
                         "floored": bool(flo[j])}
                try:
                    out[i] = (Prediction(float(mlat[j]), key, comps), PREDICTOR_MEMBOUND,
                              ["floored"] if flo[j] else [])
                except PredictionError as exc:
                    errors[i] = wrap(i, exc)
        if errors:
            raise errors[min(errors)]
        return out, totals

    def predict_layer(self, layer: LayerSpec):
        return self.predict_layers([layer])[0]


_PINNED: Dict[str, object] = {}


def _staged_upload(a: np.ndarray, dev):
    """Host array -> device through a reused page-locked staging buffer
    (asynchronous copy on the current stream; the caller's single
    device->host copy at the end of the pipeline orders the buffer's reuse)."""
    import torch
    key = a.dtype.str
    buf = _PINNED.get(key)
    if buf is None or buf.numel() < a.size:
        cap = max(1024, 1 << int(max(a.size, 1) - 1).bit_length())
        buf = _PINNED[key] = torch.empty(cap, dtype=torch.from_numpy(a[:0]).dtype,
                                         pin_memory=True)
    if a.size:
        buf[:a.size].numpy()[:] = a
    return buf[:max(a.size, 0)].to(dev, non_blocking=True)


def _staged_download(d) -> np.ndarray:
    """A device tensor's bytes into a reused page-locked buffer (one copy on
    the current stream, then a stream synchronize); returns a uint8 view,
    valid until the next call."""
    import torch
    nb = d.numel() * d.element_size()
    buf = _PINNED.get("down")
    if buf is None or buf.numel() < nb:
        buf = _PINNED["down"] = torch.empty(max(4096, 1 << int(max(nb, 1) - 1).bit_length()),
                                            dtype=torch.uint8, pin_memory=True)
    if nb:
        buf[:nb].copy_(d.reshape(-1).view(torch.uint8), non_blocking=True)
    torch.cuda.current_stream().synchronize()
    return buf[:nb].numpy()


_PREDICTORS: Dict[tuple, tuple] = {}


def _predictor(dataset: Dataset, wm: Optional[WaveModel], floor_us: float) -> ModelPredictor:
    """The ModelPredictor of (dataset, wave model, floor), kept across calls:
    its resolver holds the staged device tables of every triple it has seen
    and its fitted membound models, so repeated predict_model calls on one
    dataset stage nothing (the reference rebuilds both per call,
    aggregate.py:178).  Keyed by object identity and checked through a weak
    reference (Dataset is immutable); bounded."""
    import weakref
    key = (id(dataset), wm, floor_us)
    hit = _PREDICTORS.get(key)
    if hit is not None and hit[0]() is dataset:
        return hit[1]
    if len(_PREDICTORS) >= 16:
        _PREDICTORS.clear()
    p = ModelPredictor(dataset, wm, floor_us)
    _PREDICTORS[key] = (weakref.ref(dataset), p)
    return p


def segment_fsum(values: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """Per-segment correctly rounded sums on the GPU (== math.fsum)."""
    from . import _device, _native
    dev = _device.device()
    v = _device.to_device(np.ascontiguousarray(values, dtype=np.float64), dev)
    o = _device.to_device(np.ascontiguousarray(offsets, dtype=np.int64), dev)
    nseg = len(offsets) - 1
    out = _device.empty(max(nseg, 0), "float64", dev)
    _native.check(_native.load().pm2l_segment_fsum(_native.ptr(v), _native.ptr(o), nseg,
                                                   _native.ptr(out), _device.stream()),
                  "pm2l_segment_fsum")
    return _device.to_numpy(out)


def predict_models(graphs: Sequence[ModelGraph], dataset: Dataset,
                   wm: Optional[WaveModel] = None,
                   membound_floor_us: float = DEFAULT_LAUNCH_FLOOR_US) -> List[ModelPrediction]:
    """predict_model over many graphs with one device batch per stage."""
    predictor = _predictor(dataset, wm, membound_floor_us)
    layers = [layer for g in graphs for layer in g.layers]
    offsets = np.zeros(len(graphs) + 1, dtype=np.int64)
    np.cumsum([len(g.layers) for g in graphs], out=offsets[1:])
    res, totals = predictor._predict_layers(layers, offsets)
    if totals is None:
        totals = np.zeros(len(graphs), np.float64)   # only when there are no layers
    out = []
    for gi, g in enumerate(graphs):
        lo, hi = int(offsets[gi]), int(offsets[gi + 1])
        per = tuple(LayerPrediction(layers[i].layer_id, res[i][0], res[i][1])
                    for i in range(lo, hi))
        flags = tuple((layers[i].layer_id, f) for i in range(lo, hi) for f in res[i][2])
        out.append(ModelPrediction(g.model_name, float(totals[gi]), per, flags))
    return out


def predict_model(graph: ModelGraph, dataset: Dataset, wm: Optional[WaveModel] = None,
                  membound_floor_us: float = DEFAULT_LAUNCH_FLOOR_US) -> ModelPrediction:
    """Predict every layer and sum exactly (aggregate.py:173-196)."""
    return predict_models([graph], dataset, wm, membound_floor_us)[0]


@dataclass(frozen=True)
class TemplateLayer:
    """One layer of a model template (the same kind for every model of a
    NAS grid): a compute family (shape per model) or a utility kernel
    (features per model)."""
    layer_id: str
    family: str
    dtype: DType
    transpose_mode: Optional[TransposeMode] = None


def predict_model_grid(template: Sequence[TemplateLayer], shapes, features, dataset: Dataset,
                       wm: Optional[WaveModel] = None,
                       membound_floor_us: float = DEFAULT_LAUNCH_FLOOR_US):
    """predict_models for a NAS grid given as arrays: ``shapes`` [n_models,
    L, 4] (batch, m, n, k; compute layers), ``features`` [n_models, L, 5]
    (utility layers; FIELD_ORDER).  Returns (per-layer latency f64[n, L],
    per-model total f64[n]) with the same values as predict_models on the
    equivalent graphs (resolution + prediction per compute layer in one
    device batch per kernel triple, pm2l_points_predict; membound batches;
    exact per-model totals, pm2l_segment_fsum).  Raises UnresolvedLayer for
    the first (model, layer) that cannot be predicted."""
    from . import _device, _native
    from .compute import _log2_extension, _shapes_u32
    pred = _predictor(dataset, wm, membound_floor_us)
    L = len(template)
    shapes = np.asarray(shapes)
    n = shapes.shape[0] if shapes.ndim == 3 else np.asarray(features).shape[0]
    by_triple: Dict[tuple, List[int]] = {}
    util: Dict[tuple, List[int]] = {}
    for l, t in enumerate(template):
        if is_utility_family(t.family):
            util.setdefault((utility_kernel_name(t.family), t.dtype), []).append(l)
        elif t.family in COMPUTE_FAMILIES:
            tr = t.transpose_mode or default_transpose(t.family)
            by_triple.setdefault((t.family, t.dtype, tr), []).append(l)
        else:
            raise UnresolvedLayer(f"layer {t.layer_id!r}: no predictor for family {t.family!r}")
    # one device pipeline (as ModelPredictor._predict_layers): one staged
    # upload per input kind, every kernel back to back on the stream (one
    # resolution + prediction batch per kernel triple, one membound batch,
    # the scatter into model-major order, the exact per-model sums), one
    # device->host copy of every output
    rows = np.arange(n, dtype=np.int64)[:, None] * L
    tri = []                     # (triple, layers, ops)
    sh_parts, posc = [], []
    for triple, ls in by_triple.items():
        tri.append((triple, ls, n * len(ls)))
        sh_parts.append(_shapes_u32(shapes[:, ls, :].reshape(-1, 4)))
        posc.append((rows + np.asarray(ls, np.int64)[None, :]).ravel())
    sh = np.concatenate(sh_parts) if sh_parts else np.zeros((0, 4), np.uint32)
    nc = len(sh)
    models, mids, posu, feats = [], [], [], []
    if util:
        f = np.asarray(features, dtype=np.float64)
        for mi, ((name, dt_), ls) in enumerate(util.items()):
            models.append(pred.membound_model(name, dt_))
            for l in ls:
                feats.append(f[:, l, :])
                mids.append(np.full(n, mi, np.int64))
                posu.append(rows[:, 0] + l)
    nu = n * sum(len(ls) for ls in util.values())
    ints = np.concatenate([sh.astype(np.int64).ravel()] + mids + posc + posu +
                          [np.arange(0, n * L + 1, L, dtype=np.int64)])
    floats = np.zeros(0, np.float64)
    if nu:
        floats = np.concatenate([np.concatenate(feats).ravel(),
                                 np.array([m.weights for m in models], np.float64).ravel(),
                                 np.array([m.intercept for m in models], np.float64),
                                 np.full(len(models), membound_floor_us, np.float64)])
    dev = _device.device()
    t = _device.torch()
    lib = _native.load()
    s = _device.stream()
    d_int = _staged_upload(ints, dev)
    d_flt = _staged_upload(floats, dev) if nu else None
    o = 4 * nc
    d_mid = d_int[o:o + nu]
    o += nu
    d_posc = d_int[o:o + nc]
    o += nc
    d_posu = d_int[o:o + nu]
    o += nu
    d_off = d_int[o:o + n + 1]
    # outputs in one f64 buffer: compute latencies, match codes (int8 in their
    # own slot), membound latencies, the model-major layer latencies, totals
    sizes = [nc, (nc + 7) // 8, nu, n * L, n]
    starts = [0]
    for z in sizes:
        starts.append(starts[-1] + int(z))
    buf = t.empty(int(starts[-1]), dtype=t.float64, device=dev)
    bp = buf.data_ptr()
    sl = lambda k: buf[starts[k]:starts[k + 1]]  # noqa: E731
    lat_d = sl(3)
    lat_d.fill_(float("nan"))
    if nc:
        d_sh = d_int[:4 * nc].to(t.int32)   # u32 descriptors (int32 bits)
        ext_c, ext_l, n_ext = _log2_extension(sh, dev)
        o = 0
        for triple, ls, k in tri:
            dt = pred.resolver.triple_tables(*triple)[4]
            _native.check(lib.pm2l_points_predict_ext(
                dt.handle, d_sh.data_ptr() + 16 * o, k, _native.ptr(ext_c), _native.ptr(ext_l),
                n_ext, bp + 8 * (starts[0] + o), 0, 0, bp + 8 * starts[1] + o, 0, 0, 0, s),
                "pm2l_points_predict_ext")
            o += k
        lat_d[d_posc] = sl(0)
    if nu:
        nf, nw, nm = 5 * nu, 5 * len(models), len(models)
        ids = d_mid.to(t.int32)
        base = d_flt.data_ptr()
        _native.check(lib.pm2l_membound_predict(
            base, ids.data_ptr(), nu, base + 8 * nf, base + 8 * (nf + nw),
            base + 8 * (nf + nw + nm), nm, bp + 8 * starts[2], 0, s), "pm2l_membound_predict")
        lat_d[d_posu] = sl(2)
    if n:
        _native.check(lib.pm2l_segment_fsum(bp + 8 * starts[3], d_off.data_ptr(), n,
                                            bp + 8 * starts[4], s), "pm2l_segment_fsum")
    host = _staged_download(buf)
    v = lambda k, dt_: host[8 * starts[k]:8 * starts[k + 1]].view(dt_)  # noqa: E731
    if nc:
        match = v(1, np.int8)[:nc]
        o = 0
        for triple, ls, k in tri:
            bad = np.nonzero(match[o:o + k] == -3)[0]
            if len(bad):
                j = int(bad[0])
                raise ValidationError(f"model {j // len(ls)} layer {template[ls[j % len(ls)]].layer_id!r}: "
                                      f"block count exceeds 2^64")
            o += k
    lat = v(3, np.float64).reshape(n, L).copy()
    totals = v(4, np.float64).copy()
    bad = np.isnan(lat)
    if bad.any():
        i, l = np.argwhere(bad)[0]
        raise UnresolvedLayer(f"model {int(i)} layer {template[l].layer_id!r}: no usable kernel "
                              f"configuration")
    # every layer is a Prediction in the reference, whose latency must be
    # finite and > 0 (core.py:383-386): a raw membound layer under a
    # non-positive floor fails there, so it fails here
    bad = ~(np.isfinite(lat) & (lat > 0))
    if bad.any():
        i, l = np.argwhere(bad)[0]
        raise ValidationError(f"model {int(i)} layer {template[l].layer_id!r}: latency_us must "
                              f"be finite and > 0, got {float(lat[i, l])!r}")
    return lat, totals
