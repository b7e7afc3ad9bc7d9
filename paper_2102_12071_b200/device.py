"""PyTorch as plumbing: device buffers, streams and host<->device copies for the
C-ABI.  No arithmetic of the hot path happens in torch."""

from __future__ import annotations

import ctypes as C

import numpy as np

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t
        _torch = t
    return _torch


def require_cuda(device: int = 0):
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
    return t.device("cuda", device)


def current_device() -> int:
    return torch().cuda.current_device()


def to_dev(a, device=None, dtype=None):
    """Host array -> contiguous CUDA tensor (fp64 unless dtype given)."""
    t = torch()
    dev = require_cuda(current_device() if device is None else device)
    if isinstance(a, t.Tensor):
        x = a.to(dev)
    else:
        x = t.from_numpy(np.ascontiguousarray(a))
        x = x.to(dev, non_blocking=False)
    if dtype is not None:
        x = x.to(dtype)
    return x.contiguous()


def mask_dev(mask, device=None):
    """Bool mask -> uint8 CUDA tensor, or None when every point is active."""
    if mask is None:
        return None
    m = np.asarray(mask, dtype=bool)
    if m.all():
        return None
    return to_dev(m.astype(np.uint8), device)


def empty(shape, device=None, dtype=None):
    t = torch()
    dev = require_cuda(current_device() if device is None else device)
    return t.empty(shape, dtype=t.float64 if dtype is None else dtype, device=dev)


def zeros(shape, device=None):
    t = torch()
    dev = require_cuda(current_device() if device is None else device)
    return t.zeros(shape, dtype=t.float64, device=dev)


def ptr(x):
    """Raw device pointer of a tensor (None stays None) for the C-ABI."""
    if x is None:
        return None
    return C.c_void_p(x.data_ptr())


def stream(x=None):
    """cudaStream_t of torch's current stream on the tensor's device."""
    t = torch()
    dev = x.device if x is not None else None
    return C.c_void_p(t.cuda.current_stream(dev).cuda_stream)


def host(x) -> np.ndarray:
    return x.detach().cpu().numpy()
