"""ctypes binding of the bmode200 C ABI (include/bmode200.h).

The library is built in-tree (``_lib/libbmode200.so``) by
``paper_1811_01566_b200.build.build()``.  There is no CPU fallback: if the
library or a CUDA device is missing, every op raises ``NativeError``.
"""

from __future__ import annotations

import ctypes
import threading
import os

from .errors import NativeError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_lib", "libbmode200.so")

BM_F32, BM_F64 = 0, 1
BM_STA, BM_PW = 0, 1
BM_NEAREST, BM_LINEAR = 0, 1
BM_RECTANGULAR, BM_HANN = 0, 1
BM_ERR_AXIS_TOO_SHORT = 4
ABI_VERSION = 4

# bm_sigproc_ws_bytes ops
SIG_ANALYTIC, SIG_ENVELOPE_PEAK, SIG_ENVELOPE_DISPLAY = 0, 1, 2

# test / tuning hooks (include/bmode200.h BM_DBG_*): name -> key
DEBUG_KEYS = {"das_kernel": 0, "das_fp": 1, "das_ft": 2, "das_fpc": 3, "das_tjc": 4,
              "das_runtime_w": 5, "das_tile": 6, "das_verbose": 7, "das_generic_tz": 8,
              "fft_path": 9, "no_fused_display": 10, "fir_one_output": 11,
              "das_prefetch": 12, "das_late_producer": 13}


class DasGeometry(ctypes.Structure):
    """Mirror of ``bm_das_geometry`` (include/bmode200.h)."""

    _fields_ = [
        ("dtype", ctypes.c_int32), ("scheme", ctypes.c_int32), ("interp", ctypes.c_int32),
        ("window", ctypes.c_int32), ("uniform", ctypes.c_int32), ("n_tx", ctypes.c_int32),
        ("n_rx", ctypes.c_int32), ("n_samples", ctypes.c_int32),
        ("n_elements", ctypes.c_int32), ("n_z", ctypes.c_int32), ("n_x", ctypes.c_int32),
        ("window_hint", ctypes.c_int32), ("t0_nonzero", ctypes.c_int32),
        ("rx_identity", ctypes.c_int32), ("window_hint_wide", ctypes.c_int32),
        ("window_hint_g4", ctypes.c_int32),
        ("speed_of_sound", ctypes.c_double), ("sampling_frequency", ctypes.c_double),
        ("elem_x", ctypes.c_void_p), ("x_pos", ctypes.c_void_p), ("z_pos", ctypes.c_void_p),
        ("tx_elements", ctypes.c_void_p), ("cos_a", ctypes.c_void_p), ("sin_a", ctypes.c_void_p),
        ("rx_map", ctypes.c_void_p), ("t0_smp", ctypes.c_void_p), ("hann", ctypes.c_void_p),
        ("span", ctypes.c_void_p), ("rx_contig", ctypes.c_int32), ("tile_ls", ctypes.c_int32),
        ("rx_table", ctypes.c_void_p), ("tx_ready", ctypes.c_void_p),
        ("tx_ready_base", ctypes.c_uint32), ("weight_pad", ctypes.c_void_p),
        ("tile_ls_nearest", ctypes.c_int32), ("window_hint_g4_nearest", ctypes.c_int32),
    ]


# every symbol declared in include/bmode200.h, with its ctypes signature
_P, _I32, _I64, _D = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
SIGNATURES = {
    "bm_das_aperture_span": ([ctypes.POINTER(DasGeometry), _D, _P, _P], ctypes.c_int),
    "bm_das_prepare": ([ctypes.POINTER(DasGeometry), _P, _P, _P, _P, _P], ctypes.c_int),
    "bm_das_select": ([ctypes.POINTER(DasGeometry), _I64], ctypes.c_int),
    "bm_das_launch_shape": ([ctypes.POINTER(DasGeometry), _I64, _I32, _P], ctypes.c_int),
    "bm_das_table_bytes": ([ctypes.POINTER(DasGeometry)], _I64),
    "bm_das_build_table": ([ctypes.POINTER(DasGeometry), _P, _P], ctypes.c_int),
    "bm_das_beamform": ([ctypes.POINTER(DasGeometry), _P, _I64, _P, _I64, _I32, _P], ctypes.c_int),
    "bm_sigproc_ws_bytes": ([_I32, _I32, _I64, _I64, _I64], _I64),
    "bm_pad_traces": ([_I32, _P, _I64, _I64, _I64, _P, _I64, _P], ctypes.c_int),
    "bm_das_beamform_range": ([ctypes.POINTER(DasGeometry), _P, _I64, _P, _I64, _I32, _I32, _I32,
                               _I32, _P], ctypes.c_int),
    "bm_analytic_signal": ([_I32, _P, _P, _I64, _I64, _I64, _P, _I64, _P], ctypes.c_int),
    "bm_envelope": ([_I32, _P, _P, _I64, _P], ctypes.c_int),
    "bm_abs": ([_I32, _P, _P, _I64, _P], ctypes.c_int),
    "bm_envelope_peak": ([_I32, _P, _P, _P, _I32, _I64, _I64, _P, _I64, _P], ctypes.c_int),
    "bm_envelope_display": ([_I32, _P, _P, _P, _P, _I32, _I64, _I64, _D, _P, _I64, _P],
                            ctypes.c_int),
    "bm_fir_filter": ([_I32, _P, _I32, _P, _I64, _I64, _I64, _P, _I32, _P], ctypes.c_int),
    "bm_sliding_moments": ([_I32, _P, _I64, _I64, _I32, _I32, _I32, _I32, _P, _P, _P, _P],
                           ctypes.c_int),
    "bm_dense_forward": ([_P, _I64, _P, _P, _I32, _I32, _P, _P], ctypes.c_int),
    "bm_quantize_u8": ([_I32, _P, _P, _I64, _P], ctypes.c_int),
    "bm_simulate_rf": ([_I32, _I32, _I32, _I32, _P, _P, _P, _P, _P, _P, _D, _D, _D, _D, _P, _I32,
                        _I32, _P, _P], ctypes.c_int),
    "bm_display_tiles": ([_I32, _P, _I32, _I64, _I64, _I64, _P, _P, _D, _P], ctypes.c_int),
    "bm_check_finite": ([_I32, _P, _I64, _P, _P], ctypes.c_int),
    "bm_signal_flag": ([_P, _I32, _P], ctypes.c_int),
    "bm_stream_write_u32": ([_P, ctypes.c_uint32, _P], ctypes.c_int),
    "bm_host_upload": ([_P, _P, _P, _P, _I32, _P, _P, _P], ctypes.c_int),
    "bm_wait_flags": ([_P, _I32, _I32, _P], ctypes.c_int),
    "bm_frame_peak": ([_I32, _P, _P, _I32, _I64, _P], ctypes.c_int),
    "bm_display": ([_I32, _P, _P, _P, _P, _I32, _I64, _D, _P], ctypes.c_int),
    "bm_dynamic_adjustment": ([_I32, _P, _P, _P, _P, _I32, _I64, _D, _P], ctypes.c_int),
    "bm_debug_set": ([_I32, _I32], ctypes.c_int),
    "bm_debug_get": ([_I32], ctypes.c_int),
    "bm_error_string": ([ctypes.c_int], ctypes.c_char_p),
    "bm_abi_version": ([], ctypes.c_int),
}

_lib = None


def load():
    """Load the library (once) and declare every exported signature."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise NativeError(-1, f"{LIB_PATH} not built; run paper_1811_01566_b200.build.build()")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = res
        _lib = lib
    return _lib


def check(code: int):
    if code != 0:
        msg = load().bm_error_string(code).decode()
        raise NativeError(code, msg)


def call(name: str, *args):
    check(getattr(load(), name)(*args))


class debug_overrides:
    """Context manager setting library test/tuning hooks (bm_debug_set), e.g.
    ``with debug_overrides(das_fp=1, das_ft=2): ...``; restores the previous
    values on exit.  The library reads no environment variables."""

    def __init__(self, **kw):
        self.kw = {DEBUG_KEYS[k]: int(v) for k, v in kw.items()}
        self.prev = {}

    def __enter__(self):
        lib = load()
        for k, v in self.kw.items():
            self.prev[k] = lib.bm_debug_set(k, v)
        return self

    def __exit__(self, *exc):
        lib = load()
        for k, v in self.prev.items():
            lib.bm_debug_set(k, v)


def workspace(nbytes: int, device):
    """Caller-owned device workspace of at least ``nbytes`` (None if 0)."""
    import torch

    if nbytes <= 0:
        return None
    return torch.empty(int(nbytes), dtype=torch.uint8, device=device)


_HAVE_CUDA = False


def require_cuda():
    global _HAVE_CUDA
    if _HAVE_CUDA:
        return
    import torch

    if not torch.cuda.is_available():
        raise NativeError(-2, "no CUDA device: the B200 path has no CPU fallback")
    _HAVE_CUDA = True


class _Same:
    __slots__ = ()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False


_SAME = _Same()


def on_device(device):
    """``torch.cuda.device(device)``, or a no-op context when ``device`` is
    already current (the common case: skips torch's device-index
    bookkeeping, several microseconds per op)."""
    import torch

    idx = device.index if isinstance(device, torch.device) else device
    if idx is None or idx == torch._C._cuda_getDevice():
        return _SAME
    return torch.cuda.device(idx)


def stream_ptr(stream=None) -> int:
    """cudaStream_t of `stream`, or of the current stream of the current
    device (read directly: torch.cuda.current_stream() costs ~10 us of
    device-index bookkeeping per call, several calls per op)."""
    import torch

    if stream is not None:
        return int(stream.cuda_stream)
    return int(torch._C._cuda_getCurrentRawStream(torch._C._cuda_getDevice()))


_streams = threading.local()


def current_stream(device=None):
    """torch's current stream object of ``device`` (default: the current
    device), looked up again only when the raw stream pointer changed --
    torch.cuda.current_stream() costs ~10 us of device-index bookkeeping."""
    import torch

    idx = device.index if isinstance(device, torch.device) else device
    if idx is None:
        idx = torch._C._cuda_getDevice()
    ptr = torch._C._cuda_getCurrentRawStream(idx)
    cache = getattr(_streams, "by_dev", None)
    if cache is None:
        cache = _streams.by_dev = {}
    st = cache.get(idx)
    if st is None or st.cuda_stream != ptr:
        st = cache[idx] = torch.cuda.current_stream(idx)
    return st


def dtype_code(dtype) -> int:
    import numpy as np

    dt = np.dtype(dtype)
    if dt == np.float32:
        return BM_F32
    if dt == np.float64:
        return BM_F64
    raise NativeError(1, f"unsupported dtype {dt}")
