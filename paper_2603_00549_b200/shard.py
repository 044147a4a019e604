"""Multi-GPU sweep sharding: one process per GPU, contiguous
batch-slab shards, no data-path collective.

Every grid point is a pure function of (point, replicated tables)
(pm2lat/_kernels.pyx:97-133), so rank r predicts the batch slab
[lo_r, hi_r) on its own GPU exactly as the reference's thread pool
predicts one slab per thread (pm2lat/backend.py:78-87; the result does not
depend on the split, tests/test_nascache.py:90-97).  The one exchange
step is an all-gather of each rank's (first unresolved flat index, count),
which reproduces the single-process UnresolvedPoint semantics
(pm2lat/nascache.py:298-306) with the GLOBAL first NaN.  Results stay
sharded unless the caller asks for them (``gather=True``: rank 0 receives
every slab, as the store writer needs).

``torch.distributed`` is the plumbing (NCCL on B200 ranks, gloo in the CPU
tests); tensors live on the GPU for NCCL and on the host for gloo.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Optional, Tuple

import numpy as np

from .errors import UnresolvedPoint

_NONE = np.iinfo(np.int64).max


def shard_bounds(n_batch: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced batch slab [lo, hi) of ``rank`` (the first
    ``n_batch % world`` ranks take one extra value)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    q, r = divmod(n_batch, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


@dataclass
class ShardResult:
    lo: int                          # this rank's batch slab [lo, hi)
    hi: int
    local: np.ndarray                # latencies of the slab, canonical order
    first_unresolved: int            # global flat index of the first NaN, -1: none
    unresolved: int                  # global NaN count
    full: Optional[np.ndarray] = None  # every slab (rank 0 with gather=True)


def _dist():
    import torch.distributed as dist
    return dist


def _tensor_device(group):
    import torch
    dist = _dist()
    return torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")


def gather_unresolved(local: np.ndarray, lo: int, inner: int, group=None) -> Tuple[int, int]:
    """All-gather of (first NaN as a global flat index, NaN count) over the
    ranks: the global first unresolved point (-1 if none) and the total."""
    import torch
    dist = _dist()
    nan = np.isnan(local)
    first = lo * inner + int(np.argmax(nan)) if nan.any() else _NONE
    dev = _tensor_device(group)
    mine = torch.tensor([first, int(nan.sum())], dtype=torch.int64, device=dev)
    world = dist.get_world_size(group)
    allv = torch.empty(2 * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allv, mine, group=group)
    allv = allv.cpu().numpy().reshape(world, 2)
    first_g = int(allv[:, 0].min())
    return (-1 if first_g == _NONE else first_g), int(allv[:, 1].sum())


def _gather_to_root(local: np.ndarray, lo: int, hi: int, n_batch: int, inner: int, group):
    """Rank 0 receives every slab (send/recv, uneven shards allowed)."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = _tensor_device(group)
    if rank != 0:
        dist.send(torch.from_numpy(np.ascontiguousarray(local)).to(dev), dst=0, group=group)
        return None
    full = np.empty(n_batch * inner, np.float64)
    full[lo * inner:hi * inner] = local
    for src in range(1, world):
        s_lo, s_hi = shard_bounds(n_batch, world, src)
        buf = torch.empty((s_hi - s_lo) * inner, dtype=torch.float64, device=dev)
        if buf.numel():
            dist.recv(buf, src=src, group=group)
        full[s_lo * inner:s_hi * inner] = buf.cpu().numpy()
    return full


def predict_sharded(prep, group=None, gather: bool = False,
                    predict: Optional[Callable[[object, int, int], np.ndarray]] = None,
                    device: int = 0) -> ShardResult:
    """Predict this rank's batch slab of ``prep`` (a PreparedGrid) and
    exchange the unresolved-point statistics.  ``predict(prep, lo, hi)``
    defaults to the GPU grid kernel on ``device``."""
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    n_batch = len(prep.grid.axes["batch"])
    inner = len(prep.grid.axes["m"]) * len(prep.grid.axes["n"]) * len(prep.grid.axes["k"])
    lo, hi = shard_bounds(n_batch, world, rank)
    if predict is None:
        from . import backend
        lat = backend.predict_grid_device(prep, b_lo=lo, b_hi=hi, device=device)
        local = lat.cpu().numpy() if lat.numel() else np.empty(0, np.float64)
    else:
        local = np.ascontiguousarray(predict(prep, lo, hi), dtype=np.float64)
    first, count = gather_unresolved(local, lo, inner, group)
    full = _gather_to_root(local, lo, hi, n_batch, inner, group) if gather else None
    return ShardResult(lo, hi, local, first, count, full)


def precompute_sharded(grid, dataset, wm, out_path, group=None, skip_unresolved: bool = False,
                       predict=None, device: int = 0):
    """nascache.precompute over the ranks of ``group``: every rank predicts
    its slab; an unresolved point aborts on EVERY rank naming the global
    first one (nascache.py:298-306); rank 0 writes the store, byte-identical
    to the single-process store.  Returns the rank's ShardResult."""
    from .nascache import PreparedGrid, point_at, write_store
    prep = PreparedGrid(dataset, grid, wm)
    res = predict_sharded(prep, group=group, gather=True, predict=predict, device=device)
    if res.unresolved and not skip_unresolved:
        b, m, n, k = point_at(grid, res.first_unresolved)
        raise UnresolvedPoint(
            f"grid point batch={b} m={m} n={n} k={k} ({grid.family}, {grid.dtype.value}, "
            f"{grid.transpose_mode.value}) has no usable kernel configuration")
    if res.full is not None:
        write_store(out_path, grid, dataset, res.full)
    return res


def topk_global(values: np.ndarray, k: int, offset: int = 0, group=None) -> Tuple[np.ndarray, np.ndarray]:
    """The k smallest of a value array sharded over the ranks (SURVEY §8e:
    all-gather of the per-rank top-k, merged by (value, global index)).
    ``values`` is this rank's slice, ``offset`` its first global index.
    Returns (global indices i64[k'], values f64[k']), k' = min(k, total),
    identical on every rank; ties go to the smaller global index and NaN
    (unresolved) never ranks."""
    import torch
    dist = _dist()
    v = np.ascontiguousarray(values, dtype=np.float64)
    ok = ~np.isnan(v)
    idx = np.nonzero(ok)[0]
    order = np.lexsort((idx, v[idx]))[:k]          # (value, index) ascending
    loc_i = idx[order] + offset
    loc_v = v[idx[order]]
    dev = _tensor_device(group)
    world = dist.get_world_size(group)
    pad_i = np.full(k, np.iinfo(np.int64).max, np.int64)
    pad_v = np.full(k, np.inf)
    pad_i[:len(loc_i)] = loc_i
    pad_v[:len(loc_v)] = loc_v
    mine = torch.from_numpy(np.concatenate([pad_v.view(np.int64), pad_i])).to(dev)
    allv = torch.empty(2 * k * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allv, mine, group=group)
    a = allv.cpu().numpy().reshape(world, 2, k)
    vals = a[:, 0, :].reshape(-1).view(np.float64)
    ids = a[:, 1, :].reshape(-1)
    keep = ids != np.iinfo(np.int64).max
    vals, ids = vals[keep], ids[keep]
    sel = np.lexsort((ids, vals))[:k]
    return ids[sel], vals[sel]
