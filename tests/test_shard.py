"""Multi-rank sweep sharding on CPU: world_size 2 over gloo.
The per-slab predictor is the C oracle (test infrastructure), so this
covers the host logic the B200 ranks run: slab bounds, the all-gather of
unresolved-point statistics (global first NaN), the gather to rank 0 and
the rank-0 store write."""

import hashlib
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from conftest import GOLDEN, dataset, golden_meta, prepared

GRIDS = {g["name"]: g for g in golden_meta()["grids"]}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_slab(prep, lo, hi):
    B, M, N, K = prep.axis_arrays()
    return oracle.grid(prep.tables(), (B[lo:hi], M, N, K), verify=False)


# global flat indices forced unresolved in the "late NaN" case (both in the
# second rank's slab of exact_mix_bf16)
LATE_NAN = (0, 0)


def _oracle_slab_late_nan(prep, lo, hi):
    out = _oracle_slab(prep, lo, hi).copy()
    inner = len(out) // max(1, hi - lo)
    for g in LATE_NAN:
        if lo * inner <= g < hi * inner:
            out[g - lo * inner] = np.nan
    return out


def _worker(rank, world, port, name, tmp, q, late=None):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_00549_b200 import shard
        from paper_2603_00549_b200.compute import WaveModel
        from paper_2603_00549_b200.errors import UnresolvedPoint
        meta = GRIDS[name]
        prep = prepared(meta)
        pred = _oracle_slab
        if late is not None:
            global LATE_NAN
            LATE_NAN = late
            pred = _oracle_slab_late_nan
        res = shard.predict_sharded(prep, gather=True, predict=pred)
        out = {"rank": rank, "lo": res.lo, "hi": res.hi, "first": res.first_unresolved,
               "count": res.unresolved, "full": res.full, "local": res.local}
        ds = dataset(meta["dataset"])
        path = os.path.join(tmp, f"store_{name}.bin")
        try:
            shard.precompute_sharded(prep.grid, ds, WaveModel(ds.device.sm_count), path,
                                     predict=pred, skip_unresolved=False)
            out["raised"] = None
        except UnresolvedPoint as exc:
            out["raised"] = str(exc)
        q.put(out)
    finally:
        dist.destroy_process_group()


def _run(name, tmp_path, world=2, late=None):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, name, str(tmp_path), q, late))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = sorted((q.get(timeout=300) for _ in procs), key=lambda o: o["rank"])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return outs


def test_shard_bounds_cover_the_batch_axis():
    from paper_2603_00549_b200.shard import shard_bounds
    for nb in (0, 1, 3, 4, 7, 16):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(nb, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nb
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


@pytest.mark.parametrize("name", ["exact_mix_bf16", "mk_grid"])
def test_two_ranks_match_single_process(name, tmp_path):
    outs = _run(name, tmp_path)
    prep = prepared(GRIDS[name])
    ref = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
    full = outs[0]["full"]
    assert outs[1]["full"] is None
    assert np.array_equal(full.view(np.uint64), ref.view(np.uint64))
    inner = len(ref) // len(prep.axis_arrays()[0])
    for o in outs:
        assert np.array_equal(o["local"].view(np.uint64), ref[o["lo"] * inner:o["hi"] * inner].view(np.uint64))
        assert o["first"] == -1 and o["count"] == 0 and o["raised"] is None
    # rank 0's store is byte-identical to the single-process writer's
    from paper_2603_00549_b200.nascache import write_store
    single = tmp_path / "single.bin"
    ds = dataset(GRIDS[name]["dataset"])
    write_store(single, prep.grid, ds, ref)
    sharded = tmp_path / f"store_{name}.bin"
    assert hashlib.sha256(sharded.read_bytes()).hexdigest() == \
        hashlib.sha256(single.read_bytes()).hexdigest()


def test_two_ranks_report_global_first_unresolved(tmp_path):
    name = "unresolved_bf16_on_fp32"
    outs = _run(name, tmp_path)
    prep = prepared(GRIDS[name])
    ref = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
    nan = np.isnan(ref)
    for o in outs:
        assert o["count"] == int(nan.sum())
        assert o["first"] == int(np.argmax(nan))
        assert o["raised"] is not None and "has no usable kernel configuration" in o["raised"]


def test_global_first_unresolved_lives_on_the_second_rank(tmp_path):
    name = "exact_mix_bf16"
    prep = prepared(GRIDS[name])
    n_b = len(prep.axis_arrays()[0])
    inner = prep.grid.cardinality // n_b
    from paper_2603_00549_b200.shard import shard_bounds
    lo1, hi1 = shard_bounds(n_b, 2, 1)
    late = (hi1 * inner - 3, lo1 * inner + inner // 2)   # both in rank 1's slab
    outs = _run(name, tmp_path, late=late)
    for o in outs:
        assert o["count"] == 2
        assert o["first"] == min(late)
        b, m, n, k = __import__("paper_2603_00549_b200.nascache", fromlist=["point_at"]).point_at(
            prep.grid, min(late))
        assert o["raised"] is not None and f"batch={b} m={m} n={n} k={k}" in o["raised"]
    assert np.isnan(outs[0]["full"][list(late)]).all()


def _topk_worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2603_00549_b200.shard import shard_bounds, topk_global
        rng = np.random.default_rng(0)
        allv = np.round(rng.uniform(1, 50, 1003), 1)    # many exact ties
        allv[rng.choice(1003, 40, replace=False)] = np.nan
        lo, hi = shard_bounds(len(allv), world, rank)
        out = {"rank": rank}
        for k in (1, 7, 64, 5000):
            ids, vals = topk_global(allv[lo:hi], k, offset=lo)
            out[k] = (ids, vals)
        q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_topk_global_merges_by_value_then_index(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_topk_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(0)
    allv = np.round(rng.uniform(1, 50, 1003), 1)
    allv[rng.choice(1003, 40, replace=False)] = np.nan
    ok = np.nonzero(~np.isnan(allv))[0]
    ref = ok[np.lexsort((ok, allv[ok]))]
    for o in outs:
        for k in (1, 7, 64, 5000):
            ids, vals = o[k]
            assert np.array_equal(ids, ref[:k])
            assert np.array_equal(vals, allv[ref[:k]])
