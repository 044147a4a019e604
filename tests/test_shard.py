"""Multi-rank sweep sharding on CPU: world_size 2 and 3 over
gloo.  The per-range predictor is the C oracle (test infrastructure), so
this covers the host logic the B200 ranks run: k-row-aligned flat ranges
(a one-value batch axis still splits), the all-gather of unresolved-point
statistics (global first NaN), the grouped send/recv gather to rank 0 and
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


def _c1_meta():
    """SURVEY §8d C1 shape: batch axis (1,), 10 x 10 x 100 (fp32 tables)."""
    from paper_2603_00549_b200.core import DType, TransposeMode
    from paper_2603_00549_b200.nascache import GridSpec
    g = GridSpec("matmul", DType.FP32, TransposeMode.NN, {
        "batch": (1,), "m": tuple(range(64, 64 + 61 * 10, 61)),
        "n": tuple(range(96, 96 + 53 * 10, 53)), "k": tuple(range(32, 32 + 163 * 100, 163))})
    return {"name": "single_batch", "dataset": "fp32", "grid": g.to_json_obj(), "sm_count": 30}


GRIDS["single_batch"] = _c1_meta()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _oracle_slab(prep, lo, hi):
    """Oracle latencies of the k-row-aligned flat range [lo, hi), assembled
    from the same row pieces the device path launches."""
    from paper_2603_00549_b200.shard import row_pieces
    B, M, N, K = prep.axis_arrays()
    nK = len(K)
    parts = [oracle.grid(prep.tables(), (B, M[m0:m1], N[n0:n1], K), b0, b1, verify=False)
             for b0, b1, m0, m1, n0, n1 in row_pieces(len(M), len(N), lo // nK, hi // nK)]
    return np.concatenate(parts) if parts else np.empty(0, np.float64)


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
               "count": res.unresolved, "full": res.full_numpy(), "local": res.local_numpy()}
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


def test_shard_bounds_cover_the_axis():
    from paper_2603_00549_b200.shard import shard_bounds
    for nb in (0, 1, 3, 4, 7, 16):
        for world in (1, 2, 3, 8):
            spans = [shard_bounds(nb, world, r) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == nb
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(h - l for l, h in spans) - min(h - l for l, h in spans) <= 1


def test_row_pieces_tile_every_row_range():
    """Every k-row range decomposes into rectangular pieces that are
    contiguous in canonical order and tile it exactly (C1's single batch
    value and C3's 28 over 8 ranks included)."""
    from paper_2603_00549_b200.shard import flat_bounds, row_pieces
    rng = np.random.default_rng(0)
    cases = [(1, 10, 10, 100), (28, 1, 1, 65472), (4, 50, 50, 1000), (3, 7, 5, 2), (2, 1, 9, 3)]
    for shape in cases:
        nB, nM, nN, nK = shape
        rows = nB * nM * nN
        spans = [(0, rows)] + [tuple(sorted(rng.integers(0, rows + 1, 2))) for _ in range(50)]
        for world in (2, 3, 8):
            spans += [tuple(x // nK for x in flat_bounds(shape, world, r)) for r in range(world)]
            sizes = [(flat_bounds(shape, world, r)[1] - flat_bounds(shape, world, r)[0]) // nK
                     for r in range(world)]
            assert max(sizes) - min(sizes) <= 1         # balanced to one k-row
        for r0, r1 in spans:
            pieces = row_pieces(nM, nN, r0, r1)
            assert len(pieces) <= 5
            r = r0
            for b0, b1, m0, m1, n0, n1 in pieces:
                assert (b0 * nM + m0) * nN + n0 == r     # starts where the last ended
                assert b1 > b0 and m1 > m0 and n1 > n0
                assert (b1 - b0 == 1 or (m0 == 0 and m1 == nM)) and (m1 - m0 == 1 or (n0 == 0 and n1 == nN))
                r += (b1 - b0) * (m1 - m0) * (n1 - n0)
            assert r == r1


@pytest.mark.parametrize("name", ["exact_mix_bf16", "mk_grid"])
def test_two_ranks_match_single_process(name, tmp_path):
    outs = _run(name, tmp_path)
    prep = prepared(GRIDS[name])
    ref = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
    full = outs[0]["full"]
    assert outs[1]["full"] is None
    assert np.array_equal(full.view(np.uint64), ref.view(np.uint64))
    for o in outs:
        assert np.array_equal(o["local"].view(np.uint64), ref[o["lo"]:o["hi"]].view(np.uint64))
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
    from paper_2603_00549_b200.shard import flat_bounds
    lo1, hi1 = flat_bounds(prep.grid.shape(), 2, 1)
    late = (hi1 - 3, lo1 + (hi1 - lo1) // 2)   # both in rank 1's range
    outs = _run(name, tmp_path, late=late)
    for o in outs:
        assert o["count"] == 2
        assert o["first"] == min(late)
        b, m, n, k = __import__("paper_2603_00549_b200.nascache", fromlist=["point_at"]).point_at(
            prep.grid, min(late))
        assert o["raised"] is not None and f"batch={b} m={m} n={n} k={k}" in o["raised"]
    assert np.isnan(outs[0]["full"][list(late)]).all()


@pytest.mark.parametrize("name,world", [("mk_grid", 3), ("attn_fp32", 2), ("parity_fp32", 3)])
def test_uneven_flat_ranges_match_single_process(name, world, tmp_path):
    """Three ranks over grids whose k-rows do not divide evenly (and a
    one-(m, n)-row attention grid): ranges are row pieces, the gathered
    result and the store equal the single process's."""
    outs = _run(name, tmp_path, world=world)
    prep = prepared(GRIDS[name])
    ref = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
    assert np.array_equal(outs[0]["full"].view(np.uint64), ref.view(np.uint64))
    nK = prep.grid.shape()[3]
    spans = [(o["lo"], o["hi"]) for o in outs]
    assert spans[0][0] == 0 and spans[-1][1] == len(ref)
    assert all(lo % nK == 0 and hi % nK == 0 for lo, hi in spans)
    for o in outs:
        assert np.array_equal(o["local"].view(np.uint64), ref[o["lo"]:o["hi"]].view(np.uint64))


def test_one_value_batch_axis_splits_over_ranks(tmp_path):
    """C1-shaped grid (batch axis (1,)): every rank gets k-rows."""
    outs = _run("single_batch", tmp_path, world=2)
    assert all(o["hi"] > o["lo"] for o in outs)
    prep = prepared(GRIDS["single_batch"])
    ref = oracle.grid(prep.tables(), prep.axis_arrays(), verify=False)
    assert np.array_equal(outs[0]["full"].view(np.uint64), ref.view(np.uint64))


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


def test_gathered_ranges_are_checked_against_their_owners_checksums():
    """the stats all-gather carries each rank's range checksum;
    rank 0 checks every gathered range against it (a corrupted or misplaced
    range is caught)."""
    import torch
    from paper_2603_00549_b200 import shard
    shape = (2, 3, 5, 7)
    world = 3
    full = torch.from_numpy(np.random.default_rng(0).random(int(np.prod(shape))))
    stats = torch.zeros(world, 4, dtype=torch.int64)
    for r in range(world):
        lo, hi = shard.flat_bounds(shape, world, r)
        stats[r, 2:] = shard._range_checksum(full[lo:hi])
    shard.verify_gathered(full, stats, shape)          # intact: passes
    bad = full.clone()
    lo1, _ = shard.flat_bounds(shape, world, 1)
    bad[lo1] = np.nextafter(bad[lo1].item(), 2.0)      # one ulp in rank 1's range
    with pytest.raises(RuntimeError, match="rank 1"):
        shard.verify_gathered(bad, stats, shape)
    # checksums are order-independent within a range but not across ranges
    swapped = full.clone()
    lo2, hi2 = shard.flat_bounds(shape, world, 2)
    swapped[lo2:hi2] = torch.flip(full[lo2:hi2], [0])
    shard.verify_gathered(swapped, stats, shape)
