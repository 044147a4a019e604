"""torch plumbing: device buffers, the current stream, host<->device hand-off.

PyTorch is only used for allocation and streams; every byte of prediction
work happens in libpm2l_b200.so kernels.
"""

from __future__ import annotations

import numpy as np

from . import _native
from .errors import BackendUnavailable

_DT = None


def torch():
    import torch as _t
    return _t


def device(index: int = 0):
    t = torch()
    if not t.cuda.is_available():
        raise BackendUnavailable("torch sees no CUDA device: the B200 build has no CPU fallback")
    _native.require_gpu()
    return t.device("cuda", index)


def to_device(a: np.ndarray, dev):
    """Copy a host array to the device (pinned staging for larger inputs)."""
    t = torch()
    host = t.from_numpy(np.ascontiguousarray(a))
    if host.numel() * host.element_size() >= (1 << 20):
        host = host.pin_memory()
        return host.to(dev, non_blocking=True)
    return host.to(dev)


def empty(shape, dtype: str, dev):
    t = torch()
    return t.empty(shape, dtype=getattr(t, dtype), device=dev)


def stream():
    return _native.stream_handle()


def to_numpy(x) -> np.ndarray:
    return x.cpu().numpy()
