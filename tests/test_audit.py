"""SURVEY §8(f) row 4 against reference-generated goldens
(tests/golden/make_golden_audit.py): the interpolation-grid audit
(curvefit.grid_error_report, pm2lat/curvefit.py:192-219) and the
two-device partition cut scan (partition.partition_two_device,
pm2lat/partition.py:53-104).  CPU: the C oracle restatement; GPU: the
device kernels through the package API.  Bit-exact."""

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN, dataset

with open(os.path.join(GOLDEN, "audit.json")) as fh:
    AUDIT = json.load(fh)


def _curve(kernel):
    ds = dataset("fp32")
    fam, algo, tm, tn, sk = kernel
    for key, c in ds.curves.items():
        if (key.family, key.algorithm_id, key.tile_m, key.tile_n, key.split_k) == (fam, algo, tm, tn, sk):
            return c
    raise KeyError(kernel)


def _truth(rep):
    from paper_2603_00549_b200.curvefit import RationalTrend
    c = RationalTrend(*rep["abcd"])
    if rep["truth"] == "rational":
        return c
    return lambda d: c(d) * (1.0 + 1e-3 * ((d * 7919) % 13))   # make_golden_audit.wobble


def _fx(h):
    return float.fromhex(h)


@pytest.mark.parametrize("i", range(len(AUDIT["grid_error"])))
def test_oracle_grid_error_matches_reference(i):
    from paper_2603_00549_b200.curvefit import scan_dims
    rep = AUDIT["grid_error"][i]
    curve = _curve(rep["kernel"])
    dims = list(curve.dim_values())
    thrs = [s.throughput_gflops for s in curve.samples]
    stride, scans = scan_dims(dims, rep["max_points"])
    if rep["truth"] == "rational":
        err, arg = oracle.grid_error(dims, thrs, stride, rational=rep["abcd"])
    else:
        t = _truth(rep)
        vals = [t(d) for s in scans for d in s]
        off = np.concatenate([[0], np.cumsum([len(s) for s in scans])[:-1]])
        err, arg = oracle.grid_error(dims, thrs, stride, truth=vals, scan_off=off)
    for (lo, hi, e, a), ge, ga in zip(rep["intervals"], err, arg):
        assert ge.hex() == _fx(e).hex() and ga == a


@pytest.mark.parametrize("i", range(0, 100, 7))
def test_oracle_partition_matches_reference(i):
    p = AUDIT["partition"][i]
    la = [_fx(x) for x in p["lat_a"]]
    lb = [_fx(x) for x in p["lat_b"]]
    tr = None
    if p["link"]:
        s, g = p["link"]
        tr = [s * (1 + (cut % 3)) / (g * 1000.0) for cut in range(len(la) + 1)]
    sa, sb, bn, cut = oracle.partition(la, lb, tr)
    assert cut == p["cut"]
    assert sa[cut].hex() == _fx(p["stage_a"]).hex()
    assert sb[cut].hex() == _fx(p["stage_b"]).hex()
    assert bn[cut].hex() == _fx(p["bottleneck"]).hex()


@pytest.mark.gpu
def test_grid_error_report_on_device_matches_reference(gpu):
    from paper_2603_00549_b200.curvefit import grid_error_report
    for rep in AUDIT["grid_error"]:
        r = grid_error_report(_curve(rep["kernel"]), _truth(rep), max_points=rep["max_points"])
        assert r.max_rel_err.hex() == _fx(rep["max_rel_err"]).hex()
        assert r.argmax_dim == rep["argmax_dim"]
        got = [[iv.lo_dim, iv.hi_dim, iv.max_rel_err.hex(), iv.argmax_dim] for iv in r.intervals]
        want = [[lo, hi, _fx(e).hex(), a] for lo, hi, e, a in rep["intervals"]]
        assert got == want
        assert set(r.to_json_obj()) == {"max_rel_err", "argmax_dim", "intervals"}


def _fixture(la, lb):
    """The reference's two_device_fixture (tests/test_partition.py:27-44)."""
    from paper_2603_00549_b200.core import DeviceProfile, DType, LayerSpec, MemBoundFeatures, ModelGraph
    from paper_2603_00549_b200.ingest import Dataset
    from paper_2603_00549_b200.membound import MemBoundModel

    def profile(device_id):
        return DeviceProfile(device_id=device_id, max_freq_ghz=1.5, fp32_tflops=10.0,
                             dram_bw_gbs=300.0, mem_gb=8.0, l2_mb=4.0, sm_count=30,
                             cuda_cores=2560, power_w=100.0, collection_freq_mhz=1000.0)
    ma = MemBoundModel("stage", DType.FP32, (1, 0, 0, 0, 0), 0.0, "a", 0.0, 0.0)
    mb = MemBoundModel("stage", DType.FP32, (0, 1, 0, 0, 0), 0.0, "b", 0.0, 0.0)
    ds_a = Dataset(device=profile("dev-a"), curves={}, config_map=(), membound_records=(),
                   membound_models=(ma,))
    ds_b = Dataset(device=profile("dev-b"), curves={}, config_map=(), membound_records=(),
                   membound_models=(mb,))
    layers = tuple(LayerSpec(layer_id=f"l{j}", family="utility:stage", dtype=DType.FP32,
                             features=MemBoundFeatures(flops=a, int_ops=b, bytes_loaded=0,
                                                       bytes_stored=0, total_bytes_accessed=0))
                   for j, (a, b) in enumerate(zip(la, lb)))
    return ModelGraph(model_name="pipeline", layers=layers), ds_a, ds_b


@pytest.mark.gpu
def test_partition_two_device_on_device_matches_reference(gpu):
    from paper_2603_00549_b200.partition import link_transfer, partition_two_device, throughput_estimate
    for p in AUDIT["partition"]:
        la = [_fx(x) for x in p["lat_a"]]
        lb = [_fx(x) for x in p["lat_b"]]
        graph, ds_a, ds_b = _fixture(la, lb)
        tr = None
        if p["link"]:
            s, g = p["link"]
            tr = link_transfer(lambda cut, s=s: s * (1 + (cut % 3)), g)
        plan = partition_two_device(graph, ds_a, ds_b, transfer_us=tr)
        assert plan.cut_after_layer_index == p["cut"]
        assert plan.stage_a_us.hex() == _fx(p["stage_a"]).hex()
        assert plan.stage_b_us.hex() == _fx(p["stage_b"]).hex()
        assert plan.bottleneck_us.hex() == _fx(p["bottleneck"]).hex()
        assert float(plan.transfer_us).hex() == _fx(p["transfer"]).hex()
        assert throughput_estimate(plan, 3) == plan.stage_a_us + plan.stage_b_us + 2 * plan.bottleneck_us


@pytest.mark.gpu
def test_partition_identical_devices_cut_in_middle(gpu):
    """reference tests/test_partition.py:61-66"""
    from paper_2603_00549_b200.partition import partition_two_device
    for n_layers in (4, 5, 8, 9):
        graph, ds_a, ds_b = _fixture([10.0] * n_layers, [10.0] * n_layers)
        plan = partition_two_device(graph, ds_a, ds_b)
        assert plan.cut_after_layer_index == n_layers // 2
        assert plan.bottleneck_us == -(-n_layers // 2) * 10.0
