"""Host <-> device helpers (torch is only the allocator/stream layer)."""

from __future__ import annotations

import threading
import warnings

import numpy as np

from .types import _is_torch


# numpy arrays at least this large go through a pinned staging buffer: a
# host memcpy into page-locked memory plus a DMA at the link's full rate beats
# the driver's pageable path (~19 vs ~55 GB/s H2D on the B200 box for an
# 11.5 MB cfg2 frame)
_STAGE_MIN_BYTES = 1 << 20
_stage = threading.local()


def _staged_h2d(src, device):
    """Copy a contiguous CPU tensor to ``device`` through the per-thread
    pinned staging buffers; the copy is enqueued on the current stream."""
    import torch

    from . import _native as N

    out = torch.empty(src.shape, dtype=src.dtype, device=device)
    staged_copy_into(src, out, N.current_stream(device))
    return out


def staged_copy_into(src, dst, stream, splits=None, counter=None, values=None):
    """Copy a CPU tensor or numpy array into the device tensor ``dst`` (same
    numel) through one of two per-thread pinned staging buffers, enqueued on
    ``stream`` by bm_host_upload (multi-threaded streaming-store host copy,
    then the DMA, piece by piece); returns the event that follows the last
    DMA.  ``splits``: increasing end offsets (elements) of the pieces, else
    four for >= 4 MB.  ``counter``/``values``: device uint32 progress word
    and the value stored behind each piece (bm_stream_write_u32)."""
    import ctypes

    import torch

    from . import _native as N

    pool = getattr(_stage, "pool", None)
    if pool is None:
        pool = _stage.pool = {"bufs": [None, None], "events": [None, None], "next": 0}
    i = pool["next"]
    pool["next"] ^= 1
    if isinstance(src, np.ndarray):  # read straight from the array (no torch view)
        src = np.ascontiguousarray(src)
        esz, n, src_ptr = src.itemsize, src.size, src.ctypes.data
    else:
        src = src.contiguous()
        esz, n, src_ptr = src.element_size(), src.numel(), src.data_ptr()
    nbytes = n * esz
    if nbytes != dst.numel() * dst.element_size() or not dst.is_contiguous():
        raise ValueError("staged_copy_into: destination must be contiguous and as large as "
                         "the source")
    buf = pool["bufs"][i]
    if buf is None or buf.numel() < nbytes:
        buf = pool["bufs"][i] = torch.empty(max(nbytes, 2 * (buf.numel() if buf is not None else 0)),
                                            dtype=torch.uint8, pin_memory=True)
        pool["events"][i] = None
    ev = pool["events"][i]
    if ev is not None:
        ev.synchronize()  # the DMA that last read this buffer has finished
    if splits is None:
        step = max(1, -(-n // 4)) if nbytes >= (4 << 20) else n
        splits = list(range(step, n, step)) + [n]
    k = len(splits)
    ends = (ctypes.c_int64 * k)(*[int(e) * esz for e in splits])
    vals = (ctypes.c_uint32 * k)(*[int(v) & 0xFFFFFFFF for v in values]) if counter else None
    N.call("bm_host_upload", dst.data_ptr(), src_ptr, buf.data_ptr(), ends, k,
           counter, vals, int(stream.cuda_stream))
    ev = torch.cuda.Event()
    ev.record(stream)
    pool["events"][i] = ev
    return ev


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
    if src.numel() * src.element_size() >= _STAGE_MIN_BYTES and torch.device(device).type == "cuda":
        return _staged_h2d(src, torch.device(device))
    return src.to(device)


def torch_dtype(np_dtype):
    import torch

    return {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64,
            np.dtype(np.complex64): torch.complex64,
            np.dtype(np.complex128): torch.complex128}[np.dtype(np_dtype)]
