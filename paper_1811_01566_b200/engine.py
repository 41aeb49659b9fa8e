"""Batched B-mode reconstruction engine (cine streams).

The reference reconstructs one observation at a time through its graph
executor (pipeline.py:355-437, driven per frame by ``benchmark``).  For
streams of frames that share one acquisition geometry -- BASELINE config 4,
"batched cine stream" -- this engine runs the same chain

    das_beamform -> analytic_signal -> envelope -> dynamic_adjustment

on a batch of frames with two launches (``bm_das_beamform`` and the fused
``bm_envelope_display``: FFT -> gain -> IFFT -> |.| -> per-frame max -> dB,
the envelope kept on chip) and, for host-resident input, overlaps
the host->device copy of chunk i+1 and the device->host copy of chunk i-1
with the reconstruction of chunk i (SURVEY §8(f) "next #1": RF ingest).

Results are identical to running ``bmode_chain`` per frame: every kernel is
per-frame independent (DAS bitwise equal to the reference; peak per frame).
"""

from __future__ import annotations

import numpy as np

from . import _native as N
from .beamform import DasPlan
from .errors import AllZeroInput, InvalidMetadata, NonPositiveRange
from .types import ApodizationSpec


class BmodeEngine:
    """Reconstruct batches of frames of one (ctx, grid) on one GPU."""

    def __init__(self, ctx, grid, apod: ApodizationSpec = ApodizationSpec(),
                 interp: str = "linear", range_db: float = 30.0, dtype=np.float32,
                 n_rx: int | None = None, device=None):
        import torch

        if not (np.isfinite(range_db) and range_db > 0):
            raise NonPositiveRange(f"range_db must be > 0, got {range_db}")
        if interp not in ("nearest", "linear"):
            raise InvalidMetadata("interp", "must be one of ('nearest', 'linear')")
        n_rx = int(n_rx if n_rx is not None else (
            ctx.rx_channel_map.shape[1] if ctx.rx_channel_map is not None else ctx.n_elements))
        self.plan = DasPlan(ctx, grid, apod, dtype, n_rx, device=device)
        self.device = self.plan.device
        self.dtype = np.dtype(dtype)
        self.tdtype = torch.float32 if self.dtype == np.float32 else torch.float64
        self.code = N.dtype_code(self.dtype)
        self.interp = interp
        self.range_db = float(range_db)
        self.frame_shape = (int(ctx.n_tx), n_rx)
        self.image_shape = self.plan.shape
        self._ws = {}
        self.launches = 0

    # ------------------------------------------------------------------ device
    def _buffers(self, n_frames: int, key="dev"):
        import torch

        cur = self._ws.get(key)
        if cur is None or cur[0] < n_frames:
            nz, nx = self.image_shape
            rf_img = torch.empty((n_frames, nz, nx), dtype=self.tdtype, device=self.device)
            peak = torch.empty(n_frames, dtype=torch.int32 if self.code == N.BM_F32 else torch.int64,
                               device=self.device)
            # written for every frame by the display kernels (no fill launch)
            status = torch.empty(n_frames, dtype=torch.int32, device=self.device)
            with torch.cuda.device(self.device):
                nb = int(N.load().bm_sigproc_ws_bytes(N.SIG_ENVELOPE_DISPLAY, self.code, n_frames,
                                                      nz, nx))
            ws = N.workspace(nb, self.device)
            cur = (n_frames, rf_img, ws, peak, status, nb)
            self._ws[key] = cur
        return cur

    def reconstruct(self, rf, out=None, stream=None, key="dev", status=None, das_events=None):
        """Device batch ``rf [F, n_tx, n_rx, n_s]`` -> display ``[F, n_z, n_x]``
        (enqueued on ``stream``; no synchronisation).  Per-frame all-zero
        status is kept for :meth:`check`."""
        import torch

        f = int(rf.shape[0])
        _, rf_img, ws, peak, st, nb = self._buffers(f, key)
        rf_img, peak = rf_img[:f], peak[:f]
        status = st[:f] if status is None else status
        if out is None:
            out = torch.empty((f,) + self.image_shape, dtype=self.tdtype, device=self.device)
        s = N.stream_ptr(stream)
        if das_events is not None:
            das_events[0].record(stream)
        self.plan.beamform_batch(rf, self.interp, out=rf_img, stream=stream)
        if das_events is not None:
            das_events[1].record(stream)
        nz, nx = self.image_shape
        with torch.cuda.device(self.device):
            N.call("bm_envelope_display", self.code, rf_img.data_ptr(), out.data_ptr(),
                   peak.data_ptr(), status.data_ptr(), f, nz, nx, self.range_db, ws.data_ptr(), nb, s)
        self.launches += 2
        if not isinstance(key, tuple):
            self._last_status = status
        return out

    def check(self):
        """Raise AllZeroInput if any frame of the last batch had no positive
        envelope sample (synchronises)."""
        st = getattr(self, "_last_status", None)
        # a device->host copy of the per-frame words (no reduction kernel)
        if st is not None and st.numel() and int(st.cpu().numpy().max()) != 0:
            raise AllZeroInput("dynamic adjustment needs a strictly positive element")

    # -------------------------------------------------------------------- host
    def pinned(self, n_frames: int, n_samples: int):
        """Pinned host buffers for a host-streamed batch: (rf_host, disp_host)."""
        import torch

        rf = torch.empty((n_frames,) + self.frame_shape + (n_samples,), dtype=self.tdtype,
                         pin_memory=True)
        disp = torch.empty((n_frames,) + self.image_shape, dtype=self.tdtype, pin_memory=True)
        return rf, disp

    def reconstruct_host(self, rf_host, disp_host=None, chunk: int = 4):
        """Host batch -> host display with copy/compute overlap.

        ``rf_host`` should be pinned (see :meth:`pinned`) for the copies to be
        asynchronous.  Chunk i+1 is uploaded on an H2D stream and chunk i-1
        downloaded on a D2H stream while chunk i is reconstructed on the
        current stream.  Returns ``disp_host`` after synchronising."""
        import torch

        if disp_host is None:
            disp_host = torch.empty((int(rf_host.shape[0]),) + self.image_shape,
                                    dtype=self.tdtype, pin_memory=True)
        self.reconstruct_host_stream([(rf_host, disp_host)], chunk=chunk)
        return disp_host

    def reconstruct_host_stream(self, batches, chunk: int = 8, on_uploaded=None):
        """A stream of host batches ``[(rf_host, disp_host), ...]`` reconstructed
        as one continuous chunk pipeline (H2D of chunk i+1 and D2H of chunk
        i-1 overlap the reconstruction of chunk i, across batch boundaries),
        synchronising once at the end.  Every batch's RF is copied in and its
        display copied out.

        ``batches`` may be a lazy iterable; ``on_uploaded(i, event)`` is called
        once batch i's H2D copies are enqueued -- the batch's host RF buffer
        may be refilled after ``event`` completes."""
        import torch

        it = iter(batches)
        first = next(it, None)
        if first is None:
            return
        n_s = int(first[0].shape[-1])
        chunk = max(1, chunk)
        nbuf = 3
        key = ("host", chunk, n_s)
        if key not in self._ws:
            bufs = [torch.empty((chunk,) + self.frame_shape + (n_s,), dtype=self.tdtype,
                                device=self.device) for _ in range(nbuf)]
            outs = [torch.empty((chunk,) + self.image_shape, dtype=self.tdtype,
                                device=self.device) for _ in range(nbuf)]
            self._ws[key] = (bufs, outs, torch.cuda.Stream(self.device),
                             torch.cuda.Stream(self.device))
        bufs, outs, h2d, d2h = self._ws[key]
        comp = torch.cuda.current_stream(self.device)
        up_done = [None] * nbuf
        comp_done = [None] * nbuf
        down_done = [None] * nbuf
        statuses = []
        i = 0

        def batches_all():
            yield first
            yield from it

        for b, (rf_host, disp_host) in enumerate(batches_all()):
            f = int(rf_host.shape[0])
            status = torch.empty(f, dtype=torch.int32, device=self.device)
            statuses.append(status)
            for lo in range(0, f, chunk):
                hi = min(f, lo + chunk)
                slot = i % nbuf
                with torch.cuda.stream(h2d):
                    if comp_done[slot] is not None:
                        h2d.wait_event(comp_done[slot])  # slot's rf buffer free again
                    bufs[slot][: hi - lo].copy_(rf_host[lo:hi], non_blocking=True)
                    up_done[slot] = torch.cuda.Event()
                    up_done[slot].record(h2d)
                comp.wait_event(up_done[slot])
                if down_done[slot] is not None:
                    comp.wait_event(down_done[slot])  # slot's output buffer drained
                self.reconstruct(bufs[slot][: hi - lo], out=outs[slot][: hi - lo], stream=comp,
                                 key=("host", chunk), status=status[lo:hi])
                comp_done[slot] = torch.cuda.Event()
                comp_done[slot].record(comp)
                with torch.cuda.stream(d2h):
                    d2h.wait_event(comp_done[slot])
                    disp_host[lo:hi].copy_(outs[slot][: hi - lo], non_blocking=True)
                    down_done[slot] = torch.cuda.Event()
                    down_done[slot].record(d2h)
                i += 1
            if on_uploaded is not None:
                ev = torch.cuda.Event()
                ev.record(h2d)
                on_uploaded(b, ev)
        self._last_status = torch.cat(statuses) if len(statuses) > 1 else statuses[0]
        d2h.synchronize()
        comp.synchronize()

    def reconstruct_file(self, path, batch: int = 32, chunk: int = 8):
        """B-mode displays of every frame of a WFRF file.

        A reader thread fills two pinned host batches straight from the file
        (``WfrfReader.read_into``), so disk reads overlap the H2D copies and
        the reconstruction of the previous batch; the chunk pipeline of
        :meth:`reconstruct_host_stream` overlaps copies and compute on the
        GPU.  Returns (pinned display tensor [n_frames, n_z, n_x], context)."""
        import queue
        import threading

        import torch

        from .formats import WfrfReader

        rd = WfrfReader(path)
        try:
            if rd.frame_count == 0:
                return torch.empty((0,) + self.image_shape, dtype=self.tdtype), rd.context
            shape = tuple(rd.frame_shape)
            native = np.dtype(rd.dtype.newbyteorder("="))
            if shape[:2] != tuple(self.frame_shape) or native != self.dtype:
                from .errors import DimensionMismatch

                raise DimensionMismatch(0, f"file frames {shape} {rd.dtype} do not match the "
                                           f"engine's {self.frame_shape} {np.dtype(self.dtype)}")
            n_s = shape[2]
            disp = torch.empty((rd.frame_count,) + self.image_shape, dtype=self.tdtype,
                               pin_memory=True)
            free = queue.Queue()
            filled = queue.Queue(maxsize=2)
            for _ in range(2):
                free.put((torch.empty((batch,) + shape, dtype=self.tdtype, pin_memory=True),
                          None))
            failure = []

            def reader():
                try:
                    lo = 0
                    while lo < rd.frame_count:
                        buf, ev = free.get()
                        if ev is not None:
                            ev.synchronize()  # the GPU has copied this buffer out
                        k = rd.read_into(buf)
                        filled.put((buf, lo, k))
                        lo += k
                except Exception as exc:  # surfaced on the consumer side
                    failure.append(exc)
                filled.put(None)

            th = threading.Thread(target=reader, daemon=True)
            th.start()
            bufs_in_flight = {}

            def batches():
                b = 0
                while (item := filled.get()) is not None:
                    buf, lo, k = item
                    bufs_in_flight[b] = buf
                    b += 1
                    yield buf[:k], disp[lo:lo + k]

            def recycle(b, ev):
                free.put((bufs_in_flight.pop(b), ev))

            self.reconstruct_host_stream(batches(), chunk=chunk, on_uploaded=recycle)
            th.join()
            if failure:
                raise failure[0]
            return disp, rd.context
        finally:
            rd.close()
