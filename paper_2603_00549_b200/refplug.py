"""The reference-side binding of INTEGRATION.md, as an importable module.

The reference's only native FFI on the hot path is the Cython function
``pm2lat._kernels.predict_grid_slice`` (pm2lat/_kernels.pyx:76-133), which
``pm2lat.backend._predict_grid_compiled`` (backend.py:58-88) calls per batch
slab with the arrays of ``PreparedGrid.tables()``.  ``predict_grid_slice``
below has exactly that signature and forwards to the C ABI entry point
``pm2l_predict_grid_slice`` of libpm2l_b200.so; ``install`` swaps it in as
the backend's ``_kernels`` module, so the reference's own ``precompute`` /
``predict_grid`` run unmodified on the B200:

    import pm2lat.backend
    from paper_2603_00549_b200 import refplug
    refplug.install(pm2lat.backend)
"""

from __future__ import annotations

import types

from . import _native

_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        _LIB = _native.load()
    return _LIB


def predict_grid_slice(batch_vals, m_vals, n_vals, k_vals, b_lo, b_hi,
                       exact_keys, exact_curve, log_m, log_n, log_k, cand_curve,
                       sample_offsets, sample_dims, sample_thrs,
                       ref_dim, ref_dur, ref_thr, ref_waves,
                       tile_m, tile_n, split_k, blocks_per_wave, family_rowblock, out):
    """_kernels.predict_grid_slice (25 C-contiguous arrays / ints, writes
    ``out`` in place, returns None) on the B200."""
    P = lambda a: a.ctypes.data  # noqa: E731  (C-contiguous numpy arrays, as the caller passes)
    rc = _lib().pm2l_predict_grid_slice(
        P(batch_vals), len(batch_vals), P(m_vals), len(m_vals), P(n_vals), len(n_vals),
        P(k_vals), len(k_vals), int(b_lo), int(b_hi),
        P(exact_keys), P(exact_curve), len(exact_keys), P(log_m), P(log_n), P(log_k),
        P(cand_curve), P(sample_offsets), P(sample_dims), P(sample_thrs),
        len(sample_offsets) - 1, P(ref_dim), P(ref_dur), P(ref_thr), P(ref_waves),
        P(tile_m), P(tile_n), P(split_k), P(blocks_per_wave), P(family_rowblock), P(out))
    if rc != 0:
        raise RuntimeError(_lib().pm2l_last_error().decode())


def install(backend_module) -> types.ModuleType:
    """Point ``backend_module._kernels`` (the reference's compiled-kernel
    slot, backend.py:28-34) at this binding; returns the previous module."""
    prev = getattr(backend_module, "_kernels", None)
    backend_module._kernels = types.SimpleNamespace(predict_grid_slice=predict_grid_slice)
    return prev


__all__ = ["predict_grid_slice", "install"]
