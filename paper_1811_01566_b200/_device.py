"""Host <-> device helpers (torch is only the allocator/stream layer)."""

from __future__ import annotations

import warnings

import numpy as np

from .types import _is_torch


def to_device(a, device, dtype=None):
    """numpy or torch -> contiguous CUDA tensor (no copy if already there)."""
    import torch

    if _is_torch(a):
        t = a
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        if t.device != device:
            t = t.to(device)
        return t.contiguous()
    a = np.asarray(a)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore", UserWarning)  # read-only (frozen) numpy input
        src = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None and src.dtype != dtype:
        src = src.to(dtype)
    return src.to(device)


def torch_dtype(np_dtype):
    import torch

    return {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
            np.dtype(np.complex64): torch.complex64,
            np.dtype(np.complex128): torch.complex128}[np.dtype(np_dtype)]
