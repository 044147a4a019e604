"""Multi-GPU sweep sharding: one process per GPU, contiguous
flat-index ranges aligned to k-rows, no data-path collective.

Every grid point is a pure function of (point, replicated tables)
(pm2lat/_kernels.pyx:97-133), so a rank can predict any contiguous range
of the canonical enumeration.  The grid's k-rows -- the (b, m, n) rows of
|K| points each, ((b * nM) + m) * nN + n in canonical order -- are split
into balanced contiguous row ranges, one per rank (``row_bounds``), so a
one-value batch axis (C1) or 28 batch values over 8 ranks (C3) still
spread evenly; the reference threads only the batch axis
(pm2lat/backend.py:78-87), and its result does not depend on the split
(tests/test_nascache.py:90-97).  A row range is at most five rectangular
sub-grids (``row_pieces``), each one launch of the grid kernel on
sub-axes, written in place into the rank's device buffer.

Exchanges (NCCL over NVLink for device tensors, gloo in the CPU tests):
  * an all-gather of each rank's (first unresolved flat index, NaN count),
    computed on the device, which reproduces the single-process
    UnresolvedPoint semantics (pm2lat/nascache.py:298-306) with the GLOBAL
    first NaN;
  * optionally (``gather=True``) the results to rank 0 by one grouped
    send/recv (``batch_isend_irecv``: ncclGroupStart + ncclSend/ncclRecv,
    uneven ranges allowed) straight into rank 0's device buffer;
  * ``topk_global``: each rank's k smallest (value, global index) pairs,
    sorted on its device, all-gathered and merged on the device.
Results otherwise stay sharded on their GPUs.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Optional, Tuple

import numpy as np

from .errors import UnresolvedPoint

_NONE = np.iinfo(np.int64).max


def shard_bounds(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous, balanced range [lo, hi) of ``n`` items for ``rank`` (the
    first ``n % world`` ranks take one extra)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def row_bounds(shape: Tuple[int, int, int, int], world: int, rank: int) -> Tuple[int, int]:
    """The rank's k-row range [r0, r1) of a grid of shape (nB, nM, nN, nK)."""
    nB, nM, nN, _ = shape
    return shard_bounds(nB * nM * nN, world, rank)


def flat_bounds(shape: Tuple[int, int, int, int], world: int, rank: int) -> Tuple[int, int]:
    """The rank's flat-index range [lo, hi) (k-row aligned)."""
    r0, r1 = row_bounds(shape, world, rank)
    return r0 * shape[3], r1 * shape[3]


def row_pieces(nM: int, nN: int, r0: int, r1: int) -> List[Tuple[int, int, int, int, int, int]]:
    """The k-row range [r0, r1) as rectangular sub-grids (b0, b1, m0, m1,
    n0, n1) in canonical order: a partial (b, m) row, whole m-rows of one
    batch value, whole batch values, then the same on the way out.  Each
    piece is contiguous in the flat order and they tile the range."""
    out = []
    r, per_b = r0, nM * nN
    while r < r1:
        b, rem = divmod(r, per_b)
        m, n = divmod(rem, nN)
        left = r1 - r
        if n or left < nN:                      # inside one (b, m) row
            n1 = min(nN, n + left)
            out.append((b, b + 1, m, m + 1, n, n1))
            r += n1 - n
        elif m or left < per_b:                 # whole n-rows of batch value b
            cnt = min(nM - m, left // nN)
            out.append((b, b + 1, m, m + cnt, 0, nN))
            r += cnt * nN
        else:                                   # whole batch values
            cnt = left // per_b
            out.append((b, b + cnt, 0, nM, 0, nN))
            r += cnt * per_b
    return out


@dataclass
class ShardResult:
    lo: int                          # this rank's flat range [lo, hi)
    hi: int
    local: object                    # its latencies (torch tensor: device for NCCL, host for gloo)
    first_unresolved: int            # global flat index of the first NaN, -1: none
    unresolved: int                  # global NaN count
    full: Optional[object] = None    # every range, canonical order (rank 0 with gather=True)

    def local_numpy(self) -> np.ndarray:
        return self.local.cpu().numpy()

    def full_numpy(self) -> Optional[np.ndarray]:
        return None if self.full is None else self.full.cpu().numpy()


def _dist():
    import torch.distributed as dist
    return dist


def _tensor_device(group):
    import torch
    dist = _dist()
    return torch.device("cuda", torch.cuda.current_device()) \
        if dist.get_backend(group) == "nccl" else torch.device("cpu")


def _global(group, r: int) -> int:
    """Global rank of group rank ``r`` (send/recv peers are global ranks)."""
    return r if group is None else _dist().get_global_rank(group, r)


def predict_range_device(prep, lo: int, hi: int, out=None, device: int = 0):
    """Latencies of the flat range [lo, hi) (k-row aligned) of ``prep``'s
    grid into a CUDA float64 tensor: one grid-kernel launch per row piece,
    each on the piece's sub-axes, written in place."""
    from . import _device, _native
    g = prep.grid
    nB, nM, nN, nK = g.shape()
    if lo % max(nK, 1) or hi % max(nK, 1) or not 0 <= lo <= hi <= g.cardinality:
        raise ValueError(f"range [{lo}, {hi}) is not k-row aligned inside the grid")
    dev = _device.device(device)
    out = _device.empty(hi - lo, "float64", dev) if out is None else out
    if hi == lo:
        return out
    dt = prep.device_tables(device)
    B, M, N, K = prep.axis_arrays()
    lib = _native.load()
    s = _native.stream_handle()
    o = 0
    for b0, b1, m0, m1, n0, n1 in row_pieces(nM, nN, lo // nK, hi // nK):
        cnt = (b1 - b0) * (m1 - m0) * (n1 - n0) * nK
        _native.check(lib.pm2l_grid_predict(
            dt.handle, B.ctypes.data, nB, M.ctypes.data + 8 * m0, m1 - m0,
            N.ctypes.data + 8 * n0, n1 - n0, K.ctypes.data, nK, b0, b1,
            out.data_ptr() + 8 * o, 0, 0, 0, s), "pm2l_grid_predict")
        o += cnt
    return out


def _range_checksum(t):
    """Order-independent checksum of a float64 range: the sums of the low and
    high 32-bit halves of its bit patterns (exact in int64 below 2^31 values)
    -- the same pair wherever the bits travel, so rank 0 can check every
    gathered range against its owner's."""
    import torch
    bits = t.contiguous().view(torch.int64)
    return torch.stack([(bits & 0xFFFFFFFF).sum(), (bits >> 32 & 0xFFFFFFFF).sum()])


def _nan_stats(local, lo: int):
    """(first NaN as a global flat index or _NONE, NaN count, checksum lo,
    checksum hi) as a 4-vector on the tensor's device (no host round trip)."""
    import torch
    nan = torch.isnan(local)
    count = nan.sum()
    idx = torch.arange(local.numel(), device=local.device, dtype=torch.int64)
    first = torch.where(nan, idx + lo, torch.full_like(idx, _NONE)).min() if local.numel() \
        else torch.tensor(_NONE, device=local.device)
    return torch.cat([torch.stack([first.to(torch.int64), count.to(torch.int64)]),
                      _range_checksum(local).to(torch.int64)])


def _exchange_stats(local, lo: int, group=None):
    """All-gather of every rank's (first NaN, NaN count, checksum pair):
    one collective, a (world, 4) int64 tensor on the tensor's device."""
    import torch
    dist = _dist()
    mine = _nan_stats(local, lo)
    world = dist.get_world_size(group)
    allv = torch.empty(4 * world, dtype=torch.int64, device=mine.device)
    dist.all_gather_into_tensor(allv, mine, group=group)
    return allv.view(world, 4)


def gather_unresolved(local, lo: int, group=None) -> Tuple[int, int]:
    """All-gather of (first NaN as a global flat index, NaN count) over the
    ranks: the global first unresolved point (-1 if none) and the total."""
    allv = _exchange_stats(local, lo, group)
    first_g = int(allv[:, 0].min().item())
    return (-1 if first_g == _NONE else first_g), int(allv[:, 1].sum().item())


def verify_gathered(full, stats, shape) -> None:
    """Rank 0: every gathered range's checksum equals the one its owner
    all-gathered; raises on a mismatch."""
    world = stats.shape[0]
    for r in range(world):
        r_lo, r_hi = flat_bounds(shape, world, r)
        got = _range_checksum(full[r_lo:r_hi]).to(stats.device)
        if not bool((got == stats[r, 2:]).all()):
            raise RuntimeError(f"gathered range of rank {r} [{r_lo}, {r_hi}) fails its checksum")


def gather_to_root(local, lo: int, hi: int, shape, group=None):
    """Rank 0 receives every rank's range into one buffer on its device (one
    grouped send/recv: uneven ranges allowed); returns it on rank 0, None
    elsewhere."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if rank != 0:
        if local.numel():
            for w in dist.batch_isend_irecv([dist.P2POp(dist.isend, local.contiguous(),
                                                        _global(group, 0), group)]):
                w.wait()
        return None
    total = int(np.prod(shape))
    full = torch.empty(total, dtype=torch.float64, device=local.device)
    full[lo:hi] = local
    ops = []
    for src in range(1, world):
        s_lo, s_hi = flat_bounds(shape, world, src)
        if s_hi > s_lo:
            ops.append(dist.P2POp(dist.irecv, full[s_lo:s_hi], _global(group, src), group))
    if ops:
        for w in dist.batch_isend_irecv(ops):
            w.wait()
    return full


def predict_sharded(prep, group=None, gather: bool = False,
                    predict: Optional[Callable[[object, int, int], np.ndarray]] = None,
                    device: int = 0) -> ShardResult:
    """Predict this rank's k-row-aligned flat range of ``prep`` (a
    PreparedGrid) and exchange the unresolved-point statistics.
    ``predict(prep, lo, hi)`` (host array out) replaces the GPU kernels
    (CPU tests); by default the range is predicted on ``device``."""
    import torch
    dist = _dist()
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    shape = prep.grid.shape()
    lo, hi = flat_bounds(shape, world, rank)
    if predict is None:
        local = predict_range_device(prep, lo, hi, device=device)
    else:
        local = torch.from_numpy(np.ascontiguousarray(predict(prep, lo, hi), dtype=np.float64))
        local = local.to(_tensor_device(group))
    stats = _exchange_stats(local, lo, group)
    first_g = int(stats[:, 0].min().item())
    first, count = (-1 if first_g == _NONE else first_g), int(stats[:, 1].sum().item())
    full = gather_to_root(local, lo, hi, shape, group) if gather else None
    if full is not None:
        verify_gathered(full, stats, shape)
    return ShardResult(lo, hi, local, first, count, full)


def precompute_sharded(grid, dataset, wm, out_path, group=None, skip_unresolved: bool = False,
                       predict=None, device: int = 0):
    """nascache.precompute over the ranks of ``group``: every rank predicts
    its range; an unresolved point aborts on EVERY rank naming the global
    first one (nascache.py:298-306); rank 0 writes the store (records
    encoded on its device), byte-identical to the single-process store.
    Returns the rank's ShardResult."""
    from .nascache import PreparedGrid, point_at, write_store
    prep = PreparedGrid(dataset, grid, wm)
    res = predict_sharded(prep, group=group, gather=True, predict=predict, device=device)
    if res.unresolved and not skip_unresolved:
        b, m, n, k = point_at(grid, res.first_unresolved)
        raise UnresolvedPoint(
            f"grid point batch={b} m={m} n={n} k={k} ({grid.family}, {grid.dtype.value}, "
            f"{grid.transpose_mode.value}) has no usable kernel configuration")
    if res.full is not None:
        if res.full.is_cuda:
            from .nascache import encode_records_device
            write_store(out_path, grid, dataset, records=encode_records_device(grid, res.full))
        else:
            write_store(out_path, grid, dataset, res.full.numpy())
    return res


def topk_global(values, k: int, offset: int = 0, group=None) -> Tuple[np.ndarray, np.ndarray]:
    """The k smallest of a value array sharded over the ranks (SURVEY §8e:
    all-gather of the per-rank top-k, merged by (value, global index)).
    ``values`` is this rank's slice (torch tensor on the rank's device, or
    a host array), ``offset`` its first global index.  The selection and
    the merge run on the device (stable sorts: ties go to the smaller global
    index; NaN -- unresolved -- never ranks).  Returns (global indices
    i64[k'], values f64[k']), k' = min(k, resolved total), identical on
    every rank."""
    import torch
    dist = _dist()
    dev = _tensor_device(group)
    v = values if isinstance(values, torch.Tensor) else \
        torch.from_numpy(np.ascontiguousarray(values, dtype=np.float64))
    v = v.to(dev, torch.float64)
    world = dist.get_world_size(group)
    # stable ascending sort keeps index order on ties; NaN sorts last
    sv, si = torch.sort(v, stable=True)
    take = min(k, v.numel())
    pad_v = torch.full((k,), float("inf"), dtype=torch.float64, device=dev)
    pad_i = torch.full((k,), _NONE, dtype=torch.int64, device=dev)
    okv = sv[:take]
    ok = ~torch.isnan(okv)
    pad_v[:take] = torch.where(ok, okv, torch.full_like(okv, float("inf")))
    pad_i[:take] = torch.where(ok, si[:take].to(torch.int64) + offset,
                               torch.full_like(si[:take], _NONE, dtype=torch.int64))
    mine = torch.cat([pad_v.view(torch.int64), pad_i])
    allv = torch.empty(2 * k * world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(allv, mine, group=group)
    a = allv.view(world, 2, k)
    vals = a[:, 0, :].reshape(-1).view(torch.float64)
    ids = a[:, 1, :].reshape(-1)
    # lexicographic (value, index): stable sort by index, then by value
    o1 = torch.sort(ids, stable=True).indices
    vals, ids = vals[o1], ids[o1]
    o2 = torch.sort(vals, stable=True).indices[:k]
    vals, ids = vals[o2], ids[o2]
    keep = ids != _NONE
    return ids[keep].cpu().numpy(), vals[keep].cpu().numpy()
