"""Delay-and-Sum beamforming on the B200: drop-in for echopipe.beamform.

Same names, parameters and defaults as the reference
(/root/reference/pkg/src/echopipe/beamform.py):

* ``DasPlan(ctx, grid, apod, dtype, n_rx)`` with ``.matches(...)``
  (beamform.py:195-245) -- here it holds the *device* geometry (element and
  grid positions, tx elements / PW trig, rx map, t0, Hann table, aperture
  spans) instead of [n_elements, n_px] LUTs; the kernel rebuilds delays and
  weights on the fly with the reference's exact rounding sequence.
* ``das_beamform(frame, ctx, grid, apod, interp, n_threads, plan)``
  (beamform.py:248-296) -- ``n_threads`` is accepted and ignored (the GPU
  result is bitwise independent of any launch parameter).

Output bits equal the reference's ``das_beamform`` in f32 and f64 (pinned by
tests/test_gpu_das.py against fixtures produced by the reference).

Device policy: a numpy frame is copied to the GPU and the rf image comes
back as numpy (drop-in behaviour); a CUDA-tensor frame stays on the device
and yields a CUDA-tensor image.  The kernel is ``bm_das_beamform`` in
libbmode200.so; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _native as N
from ._device import to_device
from .errors import InvalidMetadata
from .types import ApodizationSpec, BmodeImage, RfFrame, _is_torch, validate_pair

INTERPOLATION_MODES = ("nearest", "linear")


def hann_weight_table(n_elements: int) -> np.ndarray:
    """Row M = symmetric M-point Hann window (beamform.py:48-63)."""
    tab = np.zeros((n_elements + 1, max(n_elements, 1)))
    for m_count in range(1, n_elements + 1):
        if m_count == 1:
            tab[1, 0] = 1.0
        else:
            k = np.arange(m_count)
            tab[m_count, :m_count] = 0.5 - 0.5 * np.cos(2.0 * np.pi * k / (m_count - 1))
    return tab


def active_aperture(ctx, pixel, apod: ApodizationSpec) -> np.ndarray:
    """Receive weight of every element for one pixel (beamform.py:84-119).
    Host-side helper (one pixel), same f64 gate as the kernel's span."""
    x, z = float(pixel[0]), float(pixel[1])
    elem_x = ctx.element_positions()
    n_el = elem_x.size
    if apod.f_number == 0.0:
        i0, i1 = 0, n_el - 1
    else:
        act = np.nonzero(np.abs(elem_x - x) <= z / (2.0 * apod.f_number))[0]
        i0, i1 = (int(act[0]), int(act[-1])) if act.size else (0, -1)
    w = np.zeros(n_el)
    if i1 < i0:
        return w
    if apod.window == "rectangular":
        w[i0:i1 + 1] = 1.0
    else:
        w[i0:i1 + 1] = hann_weight_table(n_el)[i1 - i0 + 1, : i1 - i0 + 1]
    return w


def _device():
    import torch

    N.require_cuda()
    return torch.device("cuda", torch.cuda.current_device())


class DasPlan:
    """Device geometry for one (ctx, grid, apod, dtype, n_rx) (beamform.py:195-245).

    Immutable after construction and safe to share between threads; the
    device buffers live on the CUDA device current at construction.
    """

    def __init__(self, ctx, grid, apod: ApodizationSpec, dtype, n_rx: int, device=None):
        import torch

        dtype = np.dtype(dtype)
        if dtype not in (np.float32, np.float64):
            raise InvalidMetadata("dtype", f"must be f32/f64, got {dtype}")
        dev = torch.device(device) if device is not None else _device()
        n_rx = int(n_rx)
        rx_map = np.ascontiguousarray(ctx.channel_elements(n_rx), dtype=np.int32)
        n_tx = int(ctx.n_tx)
        t0 = np.asarray(ctx.time_zero_offset, dtype=np.float64)
        if t0.ndim == 0:
            t0 = np.full(n_tx, float(t0))
        fs_t = dtype.type(ctx.sampling_frequency)
        # host scalars computed exactly as the reference plan does (beamform.py:230, 190-192)
        t0_smp = (fs_t * t0.astype(dtype)).astype(dtype)
        is_pw = bool(ctx.is_pw)

        def dev_t(a):
            return to_device(a, dev)

        self._bufs = {
            "elem_x": dev_t(ctx.element_positions().astype(np.float64)),
            "x_pos": dev_t(np.asarray(grid.x_positions, np.float64)),
            "z_pos": dev_t(np.asarray(grid.z_positions, np.float64)),
            "rx_map": dev_t(rx_map),
            "t0_smp": dev_t(t0_smp),
        }
        if is_pw:
            ang = np.asarray(ctx.tx_scheme.angles_rad, dtype=np.float64)
            self._bufs["cos_a"] = dev_t(np.cos(ang).astype(dtype))
            self._bufs["sin_a"] = dev_t(np.sin(ang).astype(dtype))
        else:
            self._bufs["tx_elements"] = dev_t(np.asarray(ctx.tx_scheme.tx_elements, np.int32))
        if apod.window == "hann":
            tab = hann_weight_table(ctx.n_elements).astype(dtype)
            self._bufs["hann"] = dev_t(tab)
        if apod.window == "hann" and apod.f_number > 0.0 and np.dtype(dtype) == np.float32:
            # the Hann rows zero-padded on both sides for the TMA kernel (g.weight_pad)
            n_el = ctx.n_elements
            pad = np.zeros((n_el + 1, 3 * n_el), dtype=dtype)
            pad[:, n_el:2 * n_el] = tab
            self._bufs["weight_pad"] = dev_t(pad)
        self.uniform = apod.window == "rectangular" and apod.f_number == 0.0

        g = N.DasGeometry()
        g.dtype = N.dtype_code(dtype)
        g.scheme = N.BM_PW if is_pw else N.BM_STA
        g.interp = N.BM_LINEAR
        g.window = N.BM_HANN if apod.window == "hann" else N.BM_RECTANGULAR
        g.uniform = int(self.uniform)
        g.n_tx, g.n_rx, g.n_samples = n_tx, n_rx, 1
        g.n_elements, g.n_z, g.n_x = int(ctx.n_elements), int(grid.n_z), int(grid.n_x)
        g.speed_of_sound = float(ctx.speed_of_sound)
        g.sampling_frequency = float(ctx.sampling_frequency)
        for name, buf in self._bufs.items():
            setattr(g, name, buf.data_ptr())
        if apod.f_number > 0.0:
            span = torch.empty(2 * grid.n_z * grid.n_x, dtype=torch.int32, device=dev)
            with N.on_device(dev):
                N.call("bm_das_aperture_span", ctypes.byref(g), float(apod.f_number),
                       span.data_ptr(), N.stream_ptr())
            self._bufs["span"] = span
            g.span = span.data_ptr()
        # host-side bound of the fast kernel's sample windows (bm_das_prepare)
        hx = np.ascontiguousarray(grid.x_positions, np.float64)
        hz = np.ascontiguousarray(grid.z_positions, np.float64)
        he = np.ascontiguousarray(ctx.element_positions(), np.float64)
        ht = np.ascontiguousarray(t0_smp, np.float64)
        N.call("bm_das_prepare", ctypes.byref(g), he.ctypes.data, hx.ctypes.data,
               hz.ctypes.data, ht.ctypes.data, rx_map.ctypes.data)
        self.fast_window = int(g.window_hint)
        self.tma_window = int(g.window_hint_g4)  # 4-channel TMA box width (samples)
        self._geom = g
        self.ctx, self.grid, self.apod, self.dtype, self.n_rx = ctx, grid, apod, dtype, n_rx
        self.device = dev
        self.shape = (int(grid.n_z), int(grid.n_x))
        # the geometry uploads and the span kernel ran on the stream current at
        # construction; launches on any other stream wait for this event first
        with N.on_device(dev):
            self._ready = torch.cuda.Event()
            self._ready.record()

    def matches(self, ctx, grid, apod, dtype, n_rx) -> bool:
        """Identity-keyed reuse test (beamform.py:238-245)."""
        return (self.ctx is ctx and self.grid is grid and self.apod == apod
                and self.dtype == np.dtype(dtype) and self.n_rx == n_rx)

    # one-frame launches read a per-plan receive-delay table (bm_das_build_table)
    # instead of rebuilding every CTA's delays; built lazily on the first such
    # launch, when it fits this share of the free device memory
    TABLE_MAX_FRAMES = 2
    TABLE_MEM_SHARE = 0.25
    # a host frame's copy travels in this many transmit groups, the one DAS
    # launch reading each group as it lands (beamform_host)
    HOST_PIECES = 4

    @property
    def torch_dtype(self):
        import torch

        return torch.float32 if self.dtype == np.float32 else torch.float64

    def host_overlap_ok(self, n_samples: int) -> bool:
        """beamform_host applies: trace rows already 16-B aligned (no padding
        copy, which would read the frame before it lands)."""
        return self._padded(n_samples, True) == int(n_samples)

    def delay_table(self, build: bool = True):
        """The plan's device receive-delay table (the role of the reference
        DasPlan's d_rx LUT, beamform.py:211-216, in the TMA kernel's tile
        order; n_elements x n_px f32), or None."""
        import torch

        tab = getattr(self, "_table", None)
        if tab is not None or not build:
            return tab
        if getattr(self, "_table_refused", False):
            return None
        nb = int(N.load().bm_das_table_bytes(ctypes.byref(self._geom)))
        free = torch.cuda.mem_get_info(self.device)[0]
        if nb <= 0 or nb > self.TABLE_MEM_SHARE * free:
            self._table_refused = True
            return None
        tab = torch.empty(nb // 4, dtype=torch.float32, device=self.device)
        with N.on_device(self.device):
            if self._ready is not None:
                torch.cuda.current_stream().wait_event(self._ready)  # geometry uploaded
            N.call("bm_das_build_table", ctypes.byref(self._geom), tab.data_ptr(), N.stream_ptr())
            ev = torch.cuda.Event()
            ev.record()
        self._table, self._ready = tab, ev
        return tab

    def geometry(self, n_samples: int, interp: str, fast: bool = True) -> N.DasGeometry:
        """A copy of the C descriptor for one launch (``fast=False`` forces the
        generic kernel, used by tests to cross-check the two paths)."""
        g = N.DasGeometry()
        ctypes.pointer(g)[0] = self._geom
        tab = getattr(self, "_table", None)
        g.rx_table = tab.data_ptr() if tab is not None and fast else None
        if not fast:
            g.window_hint = 0
        g.n_samples = int(n_samples)
        g.interp = N.BM_NEAREST if interp == "nearest" else N.BM_LINEAR
        return g

    KERNELS = {0: "generic", 5: "tma-ws", 6: "tma64"}

    def _padded(self, n_samples: int, fast: bool) -> int:
        """Trace length a launch runs with (fast paths: rows padded to 16 B)."""
        if not fast:
            return int(n_samples)
        q = 4 if self.dtype == np.float32 else 2
        return -(-int(n_samples) // q) * q

    def kernel_for(self, n_samples: int, interp: str = "linear", fast: bool = True) -> str:
        """Name of the CUDA kernel a launch with this trace length would use."""
        n_samples = self._padded(n_samples, fast)
        g = self.geometry(n_samples, interp, fast)
        stride = int(self._geom.n_tx) * int(self.n_rx) * int(n_samples)
        return self.KERNELS.get(N.load().bm_das_select(ctypes.byref(g), stride), "invalid")

    def launch_shape(self, n_samples: int, n_frames: int, interp: str = "linear") -> dict | None:
        """Launch shape of the TMA kernel for a batch of ``n_frames`` frames
        (``bm_das_launch_shape``), or None when another kernel would run.
        ``fp * ft`` frames share one pass: ``fp`` consumer warp groups read
        one TMEM delay table, each thread accumulates ``ft`` frames."""
        n_samples = self._padded(n_samples, True)
        g = self.geometry(n_samples, interp, True)
        stride = int(self._geom.n_tx) * int(self.n_rx) * int(n_samples)
        shape = (ctypes.c_int32 * 6)()
        if N.load().bm_das_launch_shape(ctypes.byref(g), stride, int(n_frames), shape) != 0:
            return None
        return dict(zip(("frames_per_cta", "fp", "ft", "channels_per_stage", "stages",
                         "window"), list(shape)))

    def beamform_batch(self, rf, interp: str = "linear", out=None, stream=None, fast=True,
                       tx_range=None, accumulate=False, tx_ready=None):
        """DAS of a device batch ``rf [F, n_tx, n_rx, n_s]`` (or one frame
        ``[n_tx, n_rx, n_s]``) into ``out [F, n_z, n_x]`` on ``stream``.
        ``tx_range=(e0, e1)`` beamforms those transmits only; ``accumulate``
        continues the sums already in ``out`` (bm_das_beamform_range).
        ``tx_ready=(counter_ptr, base)``: ``rf`` is still being copied in on
        another stream, which advances the device counter behind each landed
        transmit group (g.tx_ready, bm_stream_write_u32); the launch reads
        transmit e once the counter reaches base + e + 1."""
        import torch

        if interp not in INTERPOLATION_MODES:
            raise InvalidMetadata("interp", f"must be one of {INTERPOLATION_MODES}")
        single = rf.dim() == 3
        rfb = rf.unsqueeze(0) if single else rf
        f, n_tx, n_rx, n_s = rfb.shape
        if rfb.dtype != (torch.float32 if self.dtype == np.float32 else torch.float64):
            raise InvalidMetadata("data", "frame dtype differs from the plan dtype")
        if rfb.device != self.device:
            raise InvalidMetadata("data", f"frame on {rfb.device}, plan on {self.device}")
        if n_tx != self._geom.n_tx or n_rx != self.n_rx:
            raise InvalidMetadata("data", "frame shape differs from the plan")
        if out is None:
            out = torch.empty((f,) + self.shape, dtype=rfb.dtype, device=self.device)
        n_pad = n_s
        if fast and (n_s != self._padded(n_s, True) or not rfb.is_contiguous()):
            if tx_ready is not None:  # the padding copy would read RF still in flight
                raise ValueError("tx_ready launches need contiguous, 16-B aligned trace rows")
            # the TMA kernels want 16-B trace rows: copy into rows of a multiple
            # of 4 (f32) / 2 (f64) samples, zero tail (bm_pad_traces; bitwise
            # the same result)
            n_pad = self._padded(n_s, True)
            if rfb.stride(-1) != 1 or rfb.stride(-2) * n_rx != rfb.stride(-3) or \
                    rfb.stride(-3) * n_tx != rfb.stride(0):
                rfb = rfb.contiguous()
            padded = torch.empty((f, n_tx, n_rx, n_pad), dtype=rfb.dtype, device=self.device)
            N.call("bm_pad_traces", N.dtype_code(self.dtype), rfb.data_ptr(), rfb.stride(-2),
                   f * n_tx * n_rx, n_s, padded.data_ptr(), n_pad, N.stream_ptr(stream))
            rfb = padded
        elif not rfb.is_contiguous():
            rfb = rfb.contiguous()
        if fast and f <= self.TABLE_MAX_FRAMES:
            self.delay_table()
        g = self.geometry(n_pad, interp, fast)
        if tx_ready is not None:
            g.tx_ready, g.tx_ready_base = int(tx_ready[0]), int(tx_ready[1]) & 0xFFFFFFFF
        n_img = self.shape[0] * self.shape[1]
        if self._ready is not None:
            if self._ready.query():  # construction copies done: nothing left to order
                self._ready = None
            else:
                (stream if stream is not None else torch.cuda.current_stream(self.device)
                 ).wait_event(self._ready)
        e0, e1 = tx_range if tx_range is not None else (0, n_tx)
        for f0 in range(0, f, 65535):
            nf = min(65535, f - f0)
            N.call("bm_das_beamform_range", ctypes.byref(g),
                   rfb[f0].data_ptr(), n_tx * n_rx * n_pad,
                   out[f0].data_ptr(), n_img, nf, int(e0), int(e1), int(bool(accumulate)),
                   N.stream_ptr(stream))
        return out[0] if single else out


def _tx_chunks(n_tx: int, k: int):
    base, extra = divmod(n_tx, k)
    lo = 0
    for i in range(k):
        hi = lo + base + (1 if i < extra else 0)
        yield lo, hi
        lo = hi


_host_copy = threading.local()


def _copy_state(dev):
    """Per (thread, device): the copy stream host frames travel on and the
    device counter (uint32) its bm_stream_write_u32 stores advance.  One
    thread's calls are sequential and each call's copies start after the
    previous call's launch (wait_stream), so its counter only moves forward."""
    import torch

    by_dev = getattr(_host_copy, "by_dev", None)
    if by_dev is None:
        by_dev = _host_copy.by_dev = {}
    st = by_dev.get(dev.index)
    if st is None:
        st = by_dev[dev.index] = {"stream": torch.cuda.Stream(dev),
                                  "counter": torch.zeros(1, dtype=torch.int32, device=dev),
                                  "base": 0}
    return st


def beamform_host(plan: DasPlan, data, interp: str = "linear", pieces: int | None = None,
                  out=None):
    """One HOST frame (numpy, [n_tx, n_rx, n_s]) -> device rf image, the
    frame's host->device copy overlapping its own Delay-and-Sum (SURVEY
    8(f) #1): the copy runs on a copy stream in ``pieces`` transmit groups,
    each followed by a stream-ordered store of the landed-transmit count
    (bm_stream_write_u32), and ONE launch -- issued once every piece is
    enqueued, so no exception can strand it -- reads transmit e as soon as
    the count passes it (g.tx_ready).  The launch is the same kernel over
    the same data, so the bits equal a launch on the resident frame.
    ``out``: optional [1, n_z, n_x] destination, e.g. pinned host memory the
    kernel then writes over the bus."""
    import torch

    from ._device import staged_copy_into

    data = np.ascontiguousarray(data)
    if data.dtype != plan.dtype:
        raise InvalidMetadata("data", f"frame dtype {data.dtype} differs from the plan's "
                                      f"{np.dtype(plan.dtype)}")
    if data.ndim != 3 or data.shape[0] != plan._geom.n_tx or data.shape[1] != plan.n_rx:
        raise InvalidMetadata("data", f"frame shape {data.shape} does not match the plan")
    n_tx, n_rx, n_s = data.shape
    pieces = max(1, min(int(pieces or plan.HOST_PIECES), n_tx))
    dev = plan.device
    st = _copy_state(dev)
    cs, comp = st["stream"], N.current_stream(dev)
    # a buffer per call (plans are shared between threads); the copy stream
    # writes it only after the allocating stream's earlier work
    rf = torch.empty((1, n_tx, n_rx, n_s), dtype=plan.torch_dtype, device=dev)
    if out is None:
        out = torch.empty((1,) + plan.shape, dtype=plan.torch_dtype, device=dev)
    cs.wait_stream(comp)
    base = st["base"]
    st["base"] = (base + n_tx) & 0xFFFFFFFF
    ctr = st["counter"].data_ptr()
    bounds = list(_tx_chunks(n_tx, pieces))
    done = staged_copy_into(data, rf, cs,
                            splits=[e1 * n_rx * n_s for _, e1 in bounds], counter=ctr,
                            values=[base + e1 for _, e1 in bounds])
    plan.beamform_batch(rf, interp, out=out, stream=comp, tx_ready=(ctr, base))
    comp.wait_event(done)  # later users of rf on comp (its reuse) follow the copy
    return out[0]


def das_beamform(frame: RfFrame, ctx, grid, apod: ApodizationSpec = ApodizationSpec(),
                 interp: str = "linear", n_threads: int | None = None,
                 plan: DasPlan | None = None) -> BmodeImage:
    """Delay-and-Sum the frame onto the grid; returns an rf-stage image
    (beamform.py:248-296).  Computation runs in the frame's dtype."""
    if interp not in INTERPOLATION_MODES:
        raise InvalidMetadata("interp", f"must be one of {INTERPOLATION_MODES}")
    validate_pair(frame, ctx)
    dtype = np.dtype(frame.dtype)
    if plan is None or not plan.matches(ctx, grid, apod, dtype, frame.n_rx):
        plan = DasPlan(ctx, grid, apod, dtype, frame.n_rx)
    host = not _is_torch(frame.data)
    if host and plan.host_overlap_ok(frame.n_samples):
        import torch

        # the upload overlaps the DAS, which writes the image straight into
        # pinned host memory (numpy in -> numpy out, no device-to-host copy)
        out = torch.empty((1,) + plan.shape, dtype=plan.torch_dtype, pin_memory=True)
        beamform_host(plan, frame.data, interp, out=out)
        N.current_stream(plan.device).synchronize()
        return BmodeImage(out[0].numpy(), stage="rf", grid=grid)
    img = plan.beamform_batch(to_device(frame.data, plan.device), interp)
    return BmodeImage(img.cpu().numpy() if host else img, stage="rf", grid=grid)


def das_beamform_oracle(frame: RfFrame, ctx, grid, apod: ApodizationSpec = ApodizationSpec(),
                        interp: str = "linear") -> BmodeImage:
    """The reference's semantic DAS oracle (beamform.py:299-357): f64
    delays, weights and accumulation in ascending e then j, the result cast
    to the frame's dtype.  That definition is exactly the f64 Delay-and-Sum,
    which this package runs bitwise on the GPU (the reference's own
    criterion 4, test_acceptance.py:124-177, asserts the same equality for
    its numba kernel), so the oracle is evaluated by the f64 kernel on the
    frame widened to f64 -- no Python triple loop, any size."""
    import torch

    if interp not in INTERPOLATION_MODES:
        raise InvalidMetadata("interp", f"must be one of {INTERPOLATION_MODES}")
    validate_pair(frame, ctx)
    data = frame.data
    wide = data.to(torch.float64) if _is_torch(data) else np.asarray(data, dtype=np.float64)
    img = das_beamform(RfFrame(wide), ctx, grid, apod, interp)
    out = img.data
    if np.dtype(frame.dtype) == np.float32:
        out = out.to(torch.float32) if _is_torch(out) else out.astype(np.float32)
    return BmodeImage(out, stage="rf", grid=grid)
