"""Quantitative-ultrasound hooks on the B200: a drop-in for echopipe.qus
(/root/reference/pkg/src/echopipe/qus.py), the step after the envelope
(SURVEY §8(f) next #4).

* ``sliding_moments(env, window, stride)`` -- qus.py:122-158: means of X, X^2,
  X^3 over every window placement, computed on the GPU (``bm_sliding_moments``:
  one warp per placement, compensated f64 sums).
* ``dense_forward(x, model)`` / ``estimate_hk_map`` -- qus.py:161-192: the
  fully connected moments -> (u, k) model, one warp per window on the GPU
  (``bm_dense_forward``).
* ``DenseLayer`` / ``DenseModel`` / ``MomentMaps`` / ``HkParamsMap`` and the
  model file format (``save_model`` / ``load_model``, qus.py:195-279) are host
  code with the reference's validation and ``FormatError`` offsets.

Results come back as numpy float64 arrays, as the reference returns them
(the maps are small: one value per window placement).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import DimensionMismatch, FormatError, InvalidMetadata, WindowTooLarge
from .types import _is_torch, _np_dtype

MODEL_MAGIC = "HKDM"
MODEL_VERSION = 1
ACTIVATIONS = ("relu", "identity", "softplus")
_ACT_CODE = {"relu": 0, "identity": 1, "softplus": 2}

# moment means can dip a hair below the exact m2 >= m1^2 bound in floating
# point; tolerate that much and no more (qus.py:35-37)
_MOMENT_SLACK = 1e-9


def _f64(a) -> np.ndarray:
    return np.asarray(a, dtype=np.float64)


def _check_moments(m1, m2, m3) -> None:
    """Shape agreement, m2 >= 0 and m2 - m1^2 >= -slack (qus.py:49-56)."""
    if m1.shape != m2.shape or m2.shape != m3.shape:
        raise DimensionMismatch(0, "moment maps must share one shape")
    if m2.size == 0:
        return
    if m2.min() < 0:
        raise InvalidMetadata("m2", "second moment must be >= 0")
    floor = -_MOMENT_SLACK * np.maximum(np.abs(m2), 1.0)
    if (m2 - m1 * m1 < floor).any():
        raise InvalidMetadata("m2", "variance m2 - m1^2 must be >= 0")


@dataclass(frozen=True, eq=False)
class MomentMaps:
    """E[X], E[X^2], E[X^3] on the sliding-window grid (qus.py:40-62)."""

    m1: np.ndarray
    m2: np.ndarray
    m3: np.ndarray
    window: tuple
    stride: tuple

    def __post_init__(self):
        _check_moments(self.m1, self.m2, self.m3)

    @property
    def shape(self) -> tuple:
        return self.m1.shape

    def stacked(self) -> np.ndarray:
        """(rows, cols, 3) in the order (m1, m2, m3)."""
        return np.stack((self.m1, self.m2, self.m3), axis=-1)


@dataclass(frozen=True, eq=False)
class DenseLayer:
    """Affine map W a + b followed by an activation (qus.py:65-82)."""

    weights: np.ndarray  # (out_width, in_width)
    bias: np.ndarray  # (out_width,)
    activation: str

    def __post_init__(self):
        w, b = _f64(self.weights), _f64(self.bias)
        shapes_ok = w.ndim == 2 and b.ndim == 1 and w.shape[0] == b.shape[0]
        if not shapes_ok:
            raise DimensionMismatch(0, "layer weights/bias shapes disagree")
        if not (np.isfinite(w).all() and np.isfinite(b).all()):
            raise InvalidMetadata("weights", "non-finite parameter")
        if self.activation not in ACTIVATIONS:
            raise InvalidMetadata("activation", f"must be one of {ACTIVATIONS}")
        object.__setattr__(self, "weights", w)
        object.__setattr__(self, "bias", b)

    @property
    def in_width(self) -> int:
        return int(self.weights.shape[1])

    @property
    def out_width(self) -> int:
        return int(self.weights.shape[0])


@dataclass(frozen=True, eq=False)
class DenseModel:
    """Layer stack from the 3 moments to the 2 outputs (u, k) (qus.py:85-104)."""

    layers: tuple

    def __post_init__(self):
        layers = tuple(self.layers)
        if len(layers) == 0:
            raise InvalidMetadata("layers", "model needs at least one layer")
        object.__setattr__(self, "layers", layers)
        if layers[0].in_width != 3:
            raise DimensionMismatch(0, "model input width must be 3")
        if layers[-1].out_width != 2:
            raise DimensionMismatch(0, "model output width must be 2")
        for i, (prev, cur) in enumerate(zip(layers, layers[1:]), start=1):
            if prev.out_width != cur.in_width:
                raise DimensionMismatch(i, f"layer {i} expects {cur.in_width}, "
                                           f"gets {prev.out_width}")


@dataclass(frozen=True, eq=False)
class HkParamsMap:
    """Homodyned-K estimates (u, k) per window placement (qus.py:107-119)."""

    u: np.ndarray
    k: np.ndarray
    window: tuple
    stride: tuple

    def __post_init__(self):
        if self.u.shape != self.k.shape:
            raise DimensionMismatch(0, "u and k maps must share one shape")
        if not (np.isfinite(self.u).all() and np.isfinite(self.k).all()):
            raise InvalidMetadata("u", "non-finite estimate")


def _device():
    import torch

    N.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


def _to_device_2d(env_img):
    """The envelope as a device tensor (f32 stays f32, anything else f64) --
    the kernel widens to f64 per element, as the reference's
    np.asarray(env_img, dtype=np.float64) does."""
    import torch

    from ._device import to_device

    if _is_torch(env_img):
        dev = env_img.device if env_img.is_cuda else _device()
        t = env_img
    else:
        t = np.asarray(env_img)
        dev = _device()
    dt = np.dtype(_np_dtype(t))
    if np.issubdtype(dt, np.complexfloating):
        raise InvalidMetadata("env_img", "moments expect a real image")
    tdt = torch.float32 if dt == np.float32 else torch.float64
    return to_device(t, dev, tdt).contiguous(), dev


def sliding_moments(env_img, window, stride=(1, 1)) -> MomentMaps:
    """Arithmetic means of X, X^2, X^3 over every window placement
    (qus.py:122-158).  Output grid dims are ``floor((dim - win) / stride) + 1``."""
    import torch

    shape = tuple(env_img.shape) if _is_torch(env_img) else np.shape(env_img)
    wh, ww = int(window[0]), int(window[1])
    sh, sw = int(stride[0]), int(stride[1])
    if len(shape) != 2:
        raise DimensionMismatch(len(shape), "moments expect a 2-D image")
    if sh < 1 or sw < 1:
        raise InvalidMetadata("stride", "strides must be >= 1")
    if wh < 1 or ww < 1:
        raise InvalidMetadata("window", "window dims must be >= 1")
    if wh > shape[0] or ww > shape[1]:
        raise WindowTooLarge(f"window {wh}x{ww} exceeds image {shape[0]}x{shape[1]}")
    img, dev = _to_device_2d(env_img)
    out_r, out_c = (shape[0] - wh) // sh + 1, (shape[1] - ww) // sw + 1
    m = torch.empty((3, out_r, out_c), dtype=torch.float64, device=dev)
    code = N.BM_F32 if img.dtype == torch.float32 else N.BM_F64
    with torch.cuda.device(dev):
        N.call("bm_sliding_moments", code, img.data_ptr(), shape[0], shape[1], wh, ww, sh, sw,
               m[0].data_ptr(), m[1].data_ptr(), m[2].data_ptr(), N.stream_ptr())
    m = m.cpu().numpy()
    return MomentMaps(m1=m[0], m2=m[1], m3=m[2], window=(wh, ww), stride=(sh, sw))


def _pack_model(model: DenseModel, dev):
    import torch

    params = np.concatenate([np.concatenate([l.weights.reshape(-1), l.bias])
                             for l in model.layers]).astype(np.float64)
    dims = np.array([[l.weights.shape[1], l.weights.shape[0], _ACT_CODE[l.activation]]
                     for l in model.layers], dtype=np.int32).reshape(-1)
    width = int(max(max(l.weights.shape) for l in model.layers))
    return (torch.from_numpy(params).to(dev), torch.from_numpy(dims).to(dev), width)


def _dense_device(x, model: DenseModel, dev):
    """x: device f64 (n, in_width) -> device f64 (n, out_width)."""
    import torch

    n = int(x.shape[0])
    out_w = model.layers[-1].weights.shape[0]
    y = torch.empty((n, out_w), dtype=torch.float64, device=dev)
    if n:
        params, dims, width = _pack_model(model, dev)
        with torch.cuda.device(dev):
            N.call("bm_dense_forward", x.data_ptr(), n, params.data_ptr(), dims.data_ptr(),
                   len(model.layers), width, y.data_ptr(), N.stream_ptr())
    return y


def dense_forward(x, model: DenseModel) -> np.ndarray:
    """Affine-then-activation composition over the layer stack (qus.py:170-183).

    Accepts a single 3-vector or a batch shaped (..., 3); returns outputs
    shaped (..., 2) (a plain 2-vector for a single input)."""
    import torch

    a = np.asarray(x, dtype=np.float64)
    in_w = model.layers[0].weights.shape[1]
    if a.shape[-1] != in_w:
        raise DimensionMismatch(0, f"input width must be {in_w}")
    dev = _device()
    lead = a.shape[:-1]
    xd = torch.from_numpy(np.ascontiguousarray(a.reshape(-1, in_w))).to(dev)
    y = _dense_device(xd, model, dev).cpu().numpy()
    return y.reshape(lead + (y.shape[-1],))


def estimate_hk_map(env_img, window, stride, model: DenseModel) -> HkParamsMap:
    """Per-window (u, k): the dense model applied to each window's moments
    (qus.py:186-192), both on the GPU."""
    moments = sliding_moments(env_img, window, stride)
    out = dense_forward(moments.stacked(), model)
    return HkParamsMap(u=out[..., 0], k=out[..., 1], window=moments.window,
                       stride=moments.stride)


def save_model(model: DenseModel, path) -> None:
    """Write the documented model file (qus.py:1-19, 195-207): an ASCII
    header, then each layer's row-major weights and bias as little-endian f64."""
    header = [f"{MODEL_MAGIC} {MODEL_VERSION}", f"layers {len(model.layers)}"]
    header += [f"{l.in_width} {l.out_width} {l.activation}" for l in model.layers]
    header.append("end")
    payload = b"".join(np.ascontiguousarray(a, dtype="<f8").tobytes()
                       for l in model.layers for a in (l.weights, l.bias))
    with open(path, "wb") as fh:
        fh.write(("\n".join(header) + "\n").encode("ascii") + payload)


class _ModelReader:
    """Cursor over a model file's bytes; every defect is a FormatError at
    the byte offset where it was detected (qus.py:210-279)."""

    def __init__(self, blob: bytes):
        self.blob, self.pos = blob, 0

    def fail(self, reason, offset=None):
        raise FormatError(self.pos if offset is None else offset, reason)

    def line(self) -> str:
        nl = self.blob.find(b"\n", self.pos)
        if nl < 0:
            self.fail("truncated header")
        text = self.blob[self.pos:nl].decode("ascii", errors="replace")
        self.pos = nl + 1
        return text

    def f64(self, count: int) -> np.ndarray:
        out = np.frombuffer(self.blob, dtype="<f8", count=count, offset=self.pos)
        self.pos += 8 * count
        return out.copy()

    def layer_spec(self):
        fields = self.line().split()
        if len(fields) != 3:
            self.fail("expected '<in> <out> <activation>'")
        try:
            in_w, out_w = (int(v) for v in fields[:2])
        except ValueError:
            self.fail("layer dims not integers")
        if min(in_w, out_w) < 1:
            self.fail("layer dims must be >= 1")
        if fields[2] not in ACTIVATIONS:
            self.fail(f"unknown activation {fields[2]!r}")
        return in_w, out_w, fields[2]


def load_model(path) -> DenseModel:
    """Parse a model file (qus.py:210-279); FormatError on any structural defect."""
    with open(path, "rb") as fh:
        rd = _ModelReader(fh.read())
    magic = rd.line().split()
    if len(magic) != 2 or magic[0] != MODEL_MAGIC:
        rd.fail("bad magic", 0)
    if magic[1] != str(MODEL_VERSION):
        rd.fail(f"unsupported version {magic[1]}", 0)
    count = rd.line().split()
    if len(count) != 2 or count[0] != "layers":
        rd.fail("expected 'layers <count>'")
    try:
        n_layers = int(count[1])
    except ValueError:
        rd.fail("layer count not an integer")
    if n_layers < 1:
        rd.fail("layer count must be >= 1")
    specs = [rd.layer_spec() for _ in range(n_layers)]
    if rd.line() != "end":
        rd.fail("expected 'end'")
    need = rd.pos + 8 * sum(o * i + o for i, o, _ in specs)
    layers = []
    for in_w, out_w, act in specs:
        if rd.pos + 8 * (out_w * in_w + out_w) > len(rd.blob):
            rd.fail("truncated parameter payload", len(rd.blob))
        w = rd.f64(out_w * in_w).reshape(out_w, in_w)
        layers.append(DenseLayer(weights=w, bias=rd.f64(out_w), activation=act))
    if need != len(rd.blob):
        rd.fail("trailing bytes after parameters")
    try:
        return DenseModel(tuple(layers))
    except (DimensionMismatch, InvalidMetadata) as exc:
        raise FormatError(rd.pos, f"inconsistent model: {exc}") from exc
