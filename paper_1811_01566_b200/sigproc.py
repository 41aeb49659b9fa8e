"""Envelope detection and log compression on the B200: drop-in for the hot
half of echopipe.sigproc (/root/reference/pkg/src/echopipe/sigproc.py:48-97).

* ``analytic_signal(x, axis=-1)``  -- sigproc.py:48-73 (one-sided spectrum
  doubling, same gain convention for even/odd N); complex64 for f32 input,
  complex128 otherwise, as scipy.fft returns.
* ``envelope(z)``                   -- sigproc.py:76-78.
* ``dynamic_adjustment(e, range_db)`` -- sigproc.py:81-97; returns float64
  like the reference (values computed in the input precision).
* ``FirSpec`` / ``fir_filter(x, spec, axis=-1)`` -- sigproc.py:20-45, the RF
  pre-filter: causal FIR with zero history, f64
  arithmetic and f64 result like lfilter(h, [1.0], x); kernel ``bm_fir_filter``.

Device policy as in beamform.py: numpy in -> numpy out; CUDA tensor in ->
CUDA tensor out.  Kernels: ``bm_analytic_signal``, ``bm_envelope``,
``bm_dynamic_adjustment`` (libbmode200.so).  Errors are raised before any
launch, with the reference's exception types; AllZeroInput needs the
device-side peak and is raised after one synchronisation.
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from ._device import to_device
from dataclasses import dataclass

from .errors import AllZeroInput, AxisTooShort, EmptyCoefficients, NonPositiveRange
from .types import _is_torch, _np_dtype


def _dev():
    import torch

    N.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


@dataclass(frozen=True, eq=False)
class FirSpec:
    """FIR filter taps, applied causally along the sample axis (sigproc.py:20-33)."""

    coefficients: np.ndarray

    def __post_init__(self):
        h = np.atleast_1d(np.asarray(self.coefficients, dtype=np.float64))
        if h.size < 1:
            raise EmptyCoefficients("FIR filter needs at least one coefficient")
        if not np.all(np.isfinite(h)):
            raise EmptyCoefficients("FIR coefficients must be finite")
        h = h.reshape(-1).copy()
        h.setflags(write=False)
        object.__setattr__(self, "coefficients", h)


def _fir_device(x, spec: FirSpec, axis: int, out_dtype):
    """``y[n] = sum_m h[m] x[n - m]`` along ``axis`` of a device tensor, f64
    arithmetic, result in ``out_dtype`` (torch dtype)."""
    import torch

    ax = axis % x.dim()
    n = int(x.shape[ax])
    if n < 1:
        raise AxisTooShort("filter axis must have length >= 1")
    x = x.contiguous()
    shape = tuple(x.shape)
    outer = int(np.prod(shape[:ax], dtype=np.int64))
    inner = int(np.prod(shape[ax + 1:], dtype=np.int64))
    y = torch.empty(shape, dtype=out_dtype, device=x.device)
    if x.numel():
        taps = torch.from_numpy(np.array(spec.coefficients, dtype=np.float64)).to(x.device)
        code_in = N.BM_F32 if x.dtype == torch.float32 else N.BM_F64
        code_out = N.BM_F32 if out_dtype == torch.float32 else N.BM_F64
        with N.on_device(x.device):
            N.call("bm_fir_filter", code_in, x.data_ptr(), code_out, y.data_ptr(), outer, n, inner,
                   taps.data_ptr(), int(taps.numel()), N.stream_ptr())
    return y


def fir_filter(x, spec: FirSpec, axis: int = -1):
    """Causal FIR convolution ``y[n] = sum_m h[m] * x[n - m]`` (sigproc.py:36-45).

    History before sample 0 is zero, so the output has the same length as the
    input along ``axis``.  Like ``lfilter(h, [1.0], x)`` the arithmetic and the
    result are float64 (the result type of f64 taps and a real frame)."""
    import torch

    is_t = _is_torch(x)
    if not is_t:
        x = np.asarray(x)
    if x.ndim == 0:
        x = x.reshape(1) if not is_t else x.reshape(1)
    if int(x.shape[axis]) < 1:
        raise AxisTooShort("filter axis must have length >= 1")
    dt = np.dtype(_np_dtype(x))
    if np.issubdtype(dt, np.complexfloating):
        raise ValueError("fir_filter expects a real tensor")
    dev = x.device if is_t and x.is_cuda else _dev()
    tdt = torch.float32 if dt == np.float32 else torch.float64
    xd = to_device(x, dev, tdt)
    y = _fir_device(xd, spec, axis, torch.float64)
    if is_t and x.is_cuda:
        return y
    return y.cpu().numpy()


def _real_dtype_for(a):
    dt = np.dtype(_np_dtype(a))
    if np.issubdtype(dt, np.complexfloating):
        raise ValueError("analytic_signal expects a real tensor")
    return np.dtype(np.float32) if dt in (np.float32, np.float16) else np.dtype(np.float64)


def analytic_signal(x, axis: int = -1):
    """Analytic signal of a real tensor via one-sided spectrum doubling."""
    import torch

    is_t = _is_torch(x)
    if not is_t:
        x = np.asarray(x)
    rdt = _real_dtype_for(x)
    n = int(x.shape[axis])
    if n < 2:
        raise AxisTooShort("analytic signal needs axis length >= 2")
    dev = x.device if is_t and x.is_cuda else _dev()
    tdt = torch.float32 if rdt == np.float32 else torch.float64
    xd = to_device(x, dev, tdt)
    ax = axis % xd.dim()
    shape = tuple(xd.shape)
    outer = int(np.prod(shape[:ax], dtype=np.int64))
    inner = int(np.prod(shape[ax + 1:], dtype=np.int64))
    z = torch.empty(shape + (2,), dtype=tdt, device=dev)
    if xd.numel():
        code = N.dtype_code(rdt)
        with N.on_device(dev):
            nb = int(N.load().bm_sigproc_ws_bytes(N.SIG_ANALYTIC, code, outer, n, inner))
            ws = N.workspace(nb, dev)
            N.call("bm_analytic_signal", code, xd.data_ptr(), z.data_ptr(), outer, n, inner,
                   ws.data_ptr() if ws is not None else None, nb, N.stream_ptr())
    zc = torch.view_as_complex(z)
    if is_t and x.is_cuda:
        return zc
    return zc.cpu().numpy()


def envelope(z):
    """Elementwise magnitude |z| (sigproc.py:76-78)."""
    import torch

    is_t = _is_torch(z)
    if not is_t:
        z = np.asarray(z)
    if not (z.is_complex() if is_t else np.iscomplexobj(z)):
        return _abs_device(z, is_t)
    dev = z.device if is_t and z.is_cuda else _dev()
    zd = to_device(z, dev)
    rdt = torch.float32 if zd.dtype == torch.complex64 else torch.float64
    if zd.dtype not in (torch.complex64, torch.complex128):
        zd = zd.to(torch.complex128)
    zr = torch.view_as_real(zd.contiguous())
    e = torch.empty(zd.shape, dtype=rdt, device=dev)
    with N.on_device(dev):
        N.call("bm_envelope", N.BM_F32 if rdt == torch.float32 else N.BM_F64, zr.data_ptr(),
               e.data_ptr(), zd.numel(), N.stream_ptr())
    return e if is_t and z.is_cuda else e.cpu().numpy()


def _abs_device(x, is_t):
    """|x| of a real tensor on the device (np.abs of a real envelope input)."""
    import torch

    dev = x.device if is_t and x.is_cuda else _dev()
    dt = np.dtype(_np_dtype(x))
    if dt not in (np.float32, np.float64):
        dt = np.dtype(np.float64)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    xd = to_device(x, dev, tdt)
    e = torch.empty_like(xd)
    if xd.numel():
        with N.on_device(dev):
            N.call("bm_abs", N.dtype_code(dt), xd.data_ptr(), e.data_ptr(), xd.numel(),
                   N.stream_ptr())
    return e if is_t and x.is_cuda else e.cpu().numpy()


def envelope_peak_device(x, n_frames: int, n_z: int, n_x: int):
    """Fused analytic -> |.| -> per-frame peak of device images ``x``
    ([n_frames, n_z, n_x] contiguous): returns (env, peak_bits)."""
    import torch

    code = N.BM_F32 if x.dtype == torch.float32 else N.BM_F64
    env = torch.empty_like(x)
    peak = torch.empty(n_frames, dtype=torch.int32 if code == N.BM_F32 else torch.int64,
                       device=x.device)
    with N.on_device(x.device):
        nb = int(N.load().bm_sigproc_ws_bytes(N.SIG_ENVELOPE_PEAK, code, n_frames, n_z, n_x))
        ws = N.workspace(nb, x.device)
        N.call("bm_envelope_peak", code, x.data_ptr(), env.data_ptr(), peak.data_ptr(), n_frames,
               n_z, n_x, ws.data_ptr() if ws is not None else None, nb, N.stream_ptr())
    return env, peak


def _dyn_device(e, range_db: float, peak=None, disp=None, status=None):
    """dB mapping on the device in e's precision; returns (disp, status).
    ``disp`` / ``status`` may be given, e.g. pinned host tensors the kernel
    then writes over the bus (no separate device-to-host copy)."""
    import torch

    dev = e.device
    code = N.BM_F32 if e.dtype == torch.float32 else N.BM_F64
    if disp is None:
        disp = torch.empty_like(e)
    if status is None:
        status = torch.empty(1, dtype=torch.int32, device=dev)
    with N.on_device(dev):
        if peak is None:
            peak = torch.empty(1, dtype=torch.int32 if code == N.BM_F32 else torch.int64, device=dev)
            N.call("bm_dynamic_adjustment", code, e.data_ptr(), peak.data_ptr(), disp.data_ptr(),
                   status.data_ptr(), 1, e.numel(), float(range_db), N.stream_ptr())
        else:
            N.call("bm_display", code, e.data_ptr(), peak.data_ptr(), disp.data_ptr(),
                   status.data_ptr(), 1, e.numel(), float(range_db), N.stream_ptr())
    return disp, status


def dynamic_adjustment(e, range_db: float):
    """Log-compress an envelope to display values in [0, 1] (sigproc.py:81-97).

    The per-frame peak maps to 1; anything ``range_db`` or more below the
    peak maps to 0; zero inputs map to 0.  Returns float64 like the reference.
    """
    import torch

    if not (np.isfinite(range_db) and range_db > 0):
        raise NonPositiveRange(f"range_db must be > 0, got {range_db}")
    is_t = _is_torch(e)
    if not is_t:
        e = np.asarray(e)
    if (e.numel() if is_t else e.size) == 0:
        raise AllZeroInput("dynamic adjustment needs a strictly positive element")
    dt = np.dtype(_np_dtype(e))
    rdt = torch.float32 if dt == np.float32 else torch.float64
    dev = e.device if is_t and e.is_cuda else _dev()
    ed = to_device(e, dev, rdt)
    disp, status = _dyn_device(ed.reshape(-1), range_db)
    if int(status.item()) != 0:
        raise AllZeroInput("dynamic adjustment needs a strictly positive element")
    out = disp.reshape(ed.shape).to(torch.float64)
    return out if is_t and e.is_cuda else out.cpu().numpy()
