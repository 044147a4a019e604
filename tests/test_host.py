"""Host-side logic (no GPU): dataset I/O, grid specs, table staging, store
format, C-ABI library surface, and the no-fallback guarantee."""

import hashlib
import json
import os
import re

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, ROOT, dataset, golden_meta, prepared

META = golden_meta()
GRIDS = {g["name"]: g for g in META["grids"]}


# ------------------------------------------------------------------ ingest
def test_dataset_roundtrip_and_fingerprint(tmp_path):
    from paper_2603_00549_b200.ingest import load_dataset, save_dataset
    ds = dataset("fp32_full")
    p = tmp_path / "ds.json"
    save_dataset(ds, p)
    back = load_dataset(p)
    assert back.fingerprint() == ds.fingerprint() == META["fingerprints"]["fp32_full"]
    assert len(dataset("bf16").curves) == 100 and len(dataset("fp32").curves) == 13


def test_ingest_errors(tmp_path):
    from paper_2603_00549_b200.errors import ParseError, SchemaError, ValidationError
    from paper_2603_00549_b200.ingest import dataset_to_json_obj, load_dataset
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    with pytest.raises(ParseError):
        load_dataset(bad)
    obj = dataset_to_json_obj(dataset("fp32"))
    del obj["curves"][0]["ref_waves"]
    bad.write_text(json.dumps(obj))
    with pytest.raises(SchemaError, match="ref_waves"):
        load_dataset(bad)
    obj = dataset_to_json_obj(dataset("fp32"))
    obj["curves"][0]["samples"] = obj["curves"][0]["samples"][::-1]
    bad.write_text(json.dumps(obj))
    with pytest.raises(ValidationError, match="ascending"):
        load_dataset(bad)
    obj = dataset_to_json_obj(dataset("fp32"))
    obj["schema_version"] = "2"
    bad.write_text(json.dumps(obj))
    with pytest.raises(SchemaError, match="schema_version"):
        load_dataset(bad)


def test_unknown_fields_warn(tmp_path):
    from paper_2603_00549_b200.ingest import dataset_to_json_obj, load_dataset
    obj = dataset_to_json_obj(dataset("fp32"))
    obj["device"]["extra"] = 1
    p = tmp_path / "w.json"
    p.write_text(json.dumps(obj))
    with pytest.warns(UserWarning, match="extra"):
        load_dataset(p)


def test_merge(tmp_path):
    from paper_2603_00549_b200.errors import DeviceMismatch
    from paper_2603_00549_b200.ingest import Dataset, merge_datasets
    ds = dataset("fp32")
    keys = list(ds.curves)
    a = Dataset(ds.device, {k: ds.curves[k] for k in keys[:6]}, ds.config_map[:50], ())
    b = Dataset(ds.device, {k: ds.curves[k] for k in keys[6:]}, ds.config_map[50:], ())
    assert merge_datasets(a, b).fingerprint() == ds.fingerprint()
    other = dataset("bf16")
    import dataclasses
    moved = dataclasses.replace(other.device, device_id="other")
    with pytest.raises(DeviceMismatch):
        merge_datasets(ds, Dataset(moved, {}, (), ()))


def test_model_graph_roundtrip():
    from paper_2603_00549_b200.ingest import model_graph_from_json_obj, model_graph_to_json_obj
    with open(os.path.join(GOLDEN, "models.json")) as fh:
        gold = json.load(fh)
    for m in gold["models"][:50]:
        g = model_graph_from_json_obj(m["graph"])
        assert model_graph_to_json_obj(g) == m["graph"]


# -------------------------------------------------------------------- grids
def test_gridspec_semantics():
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.errors import ValidationError
    from paper_2603_00549_b200.nascache import GridSpec, point_at
    g = GridSpec("matmul", DType.FP32, TransposeMode.NN,
                 {"batch": (2, 1), "m": (64,), "n": (64, 8), "k": (32, 64)})
    assert g.axes["batch"] == (1, 2) and g.axes["n"] == (8, 64)
    assert g.cardinality == 8 == len(list(g.iter_points()))
    assert [point_at(g, i) for i in range(8)] == list(g.iter_points())
    assert GridSpec.from_json_obj(g.to_json_obj()) == g
    assert GridSpec("matmul", DType.FP32, TransposeMode.NN, {"k": (1,)}).axes["batch"] == (1,)
    with pytest.raises(ValidationError, match="duplicate"):
        GridSpec("matmul", DType.FP32, TransposeMode.NN, {"k": (1, 1)})
    with pytest.raises(ValidationError, match="compute"):
        GridSpec("utility:softmax", DType.FP32, TransposeMode.NN, {"k": (1,)})
    with pytest.raises(ValidationError, match=">= 1"):
        GridSpec("matmul", DType.FP32, TransposeMode.NN, {"k": (0,)})
    assert GridSpec.from_json_obj({"family": "linear", "dtype": "fp32",
                                   "axes": {"k": [1]}}).transpose_mode == TransposeMode.TN


def test_prepared_tables_layout_matches_reference_contract():
    prep = prepared(GRIDS["matmul_bf16"])
    t = prep.tables()
    R, C = len(prep.records), len(prep.curve_list)
    assert (R, C) == (540, 60)
    # scan order (m, n, k, batch) — nascache.py:149
    keys = [(r.shape.m, r.shape.n, r.shape.k, r.shape.batch) for r in prep.records]
    assert keys == sorted(keys)
    assert np.all(np.diff(t["exact_keys"].astype(np.float64)) >= 0)
    assert t["sample_offsets"][-1] == len(t["sample_dims"]) == 540
    assert set(np.unique(t["log_k"])) == {float(p) for p in range(5, 14)}


def test_wide_coordinates_keep_unpacked_exact_table():
    prep = prepared(GRIDS["wide_fp32"])
    assert not prep.fast_path_ok
    assert prep.tables()["exact_coords"].shape == (len(prep.records), 4)


def test_block_overflow_guard():
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.errors import ValidationError
    from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid
    g = GridSpec("matmul", DType.FP32, TransposeMode.NN,
                 {"batch": (1 << 30,), "m": (1 << 30,), "n": (1 << 20,), "k": (64,)})
    with pytest.raises(ValidationError, match="2\\^53"):
        PreparedGrid(dataset("fp32"), g, WaveModel(30))


def test_store_writer_is_byte_identical_to_reference(tmp_path):
    """The vectorised store encoder fed with oracle latencies reproduces the
    reference's store bytes (nascache.py:308-333)."""
    from paper_2603_00549_b200.nascache import CacheStore, write_store
    from paper_2603_00549_b200.errors import MissingEntry
    for name in ("mk_grid", "attn_fp32"):
        prep = prepared(GRIDS[name])
        lat = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
        out = tmp_path / f"{name}.bin"
        write_store(out, prep.grid, prep.dataset, lat)
        assert hashlib.sha256(out.read_bytes()).hexdigest() == META["store"][name]["sha256"]
        with CacheStore(out) as st:
            for (b, m, n, k), v in list(st.iter_entries())[:20]:
                assert st.lookup(b, m, n, k) == v
            with pytest.raises(MissingEntry):
                st.lookup(10 ** 6, 1, 1, 1)
    prep = prepared(GRIDS["unresolved_bf16_on_fp32"])
    lat = np.full(prep.grid.cardinality, np.nan)
    out = tmp_path / "skip.bin"
    write_store(out, prep.grid, prep.dataset, lat)
    assert hashlib.sha256(out.read_bytes()).hexdigest() == META["store"]["unresolved_skip"]["sha256"]


def test_store_format_errors(tmp_path):
    from paper_2603_00549_b200.errors import CacheFormatError
    from paper_2603_00549_b200.nascache import CacheStore, write_store
    p = tmp_path / "bad.bin"
    p.write_bytes(b"NOPE" + b"\0" * 32)
    with pytest.raises(CacheFormatError):
        CacheStore(p)
    prep = prepared(GRIDS["mk_grid"])
    lat = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
    write_store(p, prep.grid, prep.dataset, lat)
    data = p.read_bytes()
    p.write_bytes(data[:-5])
    with pytest.raises(CacheFormatError, match="truncated"):
        CacheStore(p)


# -------------------------------------------------------------------- C ABI
def _header_functions():
    text = open(os.path.join(ROOT, "include", "pm2l.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pm2l_[a-z_0-9]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    from paper_2603_00549_b200 import _native
    lib = _native.load()
    names = _header_functions()
    assert len(names) >= 12
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_native.SIGNATURES)
    assert lib.pm2l_abi_version() == 1


def test_cpu_host_has_no_fallback():
    """Without a GPU every compute entry point fails loudly."""
    from paper_2603_00549_b200 import _native, backend
    from paper_2603_00549_b200.errors import BackendUnavailable
    if _native.device_count() > 0:
        pytest.skip("GPU present")
    prep = prepared(GRIDS["mk_grid"])
    with pytest.raises(BackendUnavailable):
        backend.predict_grid(prep)
    with pytest.raises(BackendUnavailable):
        prep.device_tables()
    assert _native.load().pm2l_predict_grid_slice(
        *([None, 0] * 4), 0, 0, None, None, 0, None, None, None, None, None, None, None, 0,
        None, None, None, None, None, None, None, None, None, None) == _native.PM2L_ERR_NODEVICE


def test_membound_fit_matches_reference_fit():
    """The on-demand OLS refit used by predict_model reproduces the
    reference's fitted weights bit for bit (same numpy/LAPACK)."""
    from conftest import golden_npz
    from paper_2603_00549_b200.aggregate import ModelPredictor
    from paper_2603_00549_b200.core import DType
    z = golden_npz("membound")
    mp = ModelPredictor(dataset("fp32_full"))
    for i, name in enumerate(("softmax", "gelu", "add")):
        m = mp.membound_model(name, DType.FP32)
        assert np.array_equal(np.array(m.weights), z["weights"][i])
        assert m.intercept == z["intercept"][i]
        assert m.max_rel_err == z["max_rel_err"][i]


def test_device_table_set_stages_every_triple_once():
    """one host build per (family, dtype, transpose) triple,
    identical to PreparedGrid.tables(); fingerprint-guarded reuse."""
    import numpy as np
    from conftest import dataset
    from paper_2603_00549_b200.compute import WaveModel
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.errors import StaleCache
    from paper_2603_00549_b200.nascache import GridSpec, PreparedGrid
    from paper_2603_00549_b200.staging import DeviceTableSet
    ds = dataset("bf16")
    st = DeviceTableSet(ds)
    fams = {t[0] for t in st.triples()}
    assert {"matmul", "linear", "batched_matmul"} <= fams
    for fam, dt, tm in st.triples():
        grid = GridSpec(fam, dt, tm, {"batch": (1, 2), "m": (64, 128), "n": (96,), "k": (32, 4096)})
        ref = PreparedGrid(ds, grid, WaveModel(ds.device.sm_count)).tables()
        got = st.host_tables(fam, dt, tm)
        assert set(ref) == set(got)
        for k in ref:
            a, b = ref[k], got[k]
            if a is None:
                assert b is None
            else:
                assert np.array_equal(np.asarray(a), np.asarray(b)), k
    st.verify(ds)
    with pytest.raises(StaleCache):
        st.verify(dataset("fp32"))
