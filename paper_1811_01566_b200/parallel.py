"""Multi-GPU partitioning of the B-mode path.

One process per GPU (torch.distributed; NCCL on GPUs, gloo in the CPU tests):

* **Independent frames** (config 4, cine streams): `frame_partition` deals
  frames to ranks; there is no data-path collective.

* **One large frame** (config 5, 2048 x 2048 STAI), `LateralSplit`: every
  rank owns a contiguous slab of image COLUMNS at all depths.  Delay-and-Sum
  is per pixel, so a rank's slab is bitwise the same columns of a one-GPU
  run, and the analytic signal runs along depth, so every FFT lane is
  rank-local.  Per frame a rank runs two of its own kernels and ONE
  collective:

    1. ``bm_das_beamform`` of its slab;
    2. ``bm_envelope_peak`` writing the slab's envelope AND its peak straight
       into the rank's send tile [envelope (n_z x w) | ... | peak bits];
    3. ``dist.gather`` of the tiles to ``dst`` (NCCL);

  and ``dst`` alone maps the stitched frame with ``bm_display_tiles`` (global
  peak = max of the tiles' peaks, read on the device).  No host
  synchronisation, no torch reductions, no concatenation copies.  AllZeroInput
  (sigproc.py:91-92) is raised on ``dst`` from the kernel's status word after
  the gather, so no rank can be left waiting in a collective.

* **One large frame, split by depth ROWS** (`RowSplit`, the north star's
  literal "image rows are split across GPUs"): each rank beamforms a band of
  rows at all columns -- bitwise the same pixels as one GPU -- but a band cuts
  every axial FFT lane, so the bands are gathered to ``dst`` (one gather of
  f32 RF rows), which runs the fused envelope + display of the whole frame
  (the same kernel as one GPU, so the same bits).

The collective and packing logic is plain torch.distributed over tensors,
so it runs (and is tested) with gloo on CPU tensors; the device kernels are
only called on CUDA tensors.
"""

from __future__ import annotations

import numpy as np

from .types import ImageGrid


def frame_partition(n_frames: int, world: int, rank: int) -> range:
    """Contiguous block of frame indices for `rank` (sizes differ by <= 1)."""
    base, extra = divmod(n_frames, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))


def column_slabs(n_x: int, world: int) -> list[tuple[int, int]]:
    """[lo, hi) column ranges, one per rank, sizes differing by <= 1 (the
    first n_x % world one wider -- the layout bm_display_tiles assumes)."""
    return [(r.start, r.stop) for r in (frame_partition(n_x, world, k) for k in range(world))]


def _peak_dtype(dtype):
    import torch

    return torch.int32 if dtype == torch.float32 else torch.int64


class LateralSplit:
    """Column-slab decomposition of one frame's image grid."""

    def __init__(self, grid, world: int, rank: int):
        self.grid, self.world, self.rank = grid, int(world), int(rank)
        self.slabs = column_slabs(grid.n_x, self.world)
        lo, hi = self.slabs[self.rank]
        if hi <= lo:
            raise ValueError(f"rank {rank} has no columns ({grid.n_x} columns, {world} ranks)")
        self.lo, self.hi = lo, hi
        self.sub_grid = ImageGrid(np.asarray(grid.x_positions)[lo:hi],
                                  np.asarray(grid.z_positions))

    @property
    def tile_stride(self) -> int:
        """Elements per tile: the widest slab's envelope plus one peak slot."""
        return self.grid.n_z * max(h - l for l, h in self.slabs) + 1

    def send_tile(self, dtype, device):
        import torch

        return torch.zeros(self.tile_stride, dtype=dtype, device=device)

    def recv_tiles(self, dtype, device):
        import torch

        return torch.zeros((self.world, self.tile_stride), dtype=dtype, device=device)

    def tile_views(self, tile):
        """(envelope [n_z, w] view, peak-bits [1] view) of this rank's tile."""
        return self.envelope_view(tile, self.rank), tile[-1:].view(_peak_dtype(tile.dtype))

    def envelope_view(self, tile, rank: int):
        lo, hi = self.slabs[rank]
        return tile[: self.grid.n_z * (hi - lo)].view(self.grid.n_z, hi - lo)

    def envelope_into_tile(self, rf_slab, tile):
        """Envelope + peak of this rank's beamformed slab [n_z, w] written in
        place into `tile` by bm_envelope_peak (CUDA)."""
        import torch

        from . import _native as N

        n_z, w = rf_slab.shape
        x = rf_slab.contiguous()
        code = N.BM_F32 if x.dtype == torch.float32 else N.BM_F64
        env, peak = self.tile_views(tile)
        with torch.cuda.device(x.device):
            nb = int(N.load().bm_sigproc_ws_bytes(N.SIG_ENVELOPE_PEAK, code, 1, n_z, w))
            ws = N.workspace(nb, x.device)
            N.call("bm_envelope_peak", code, x.data_ptr(), env.data_ptr(), peak.data_ptr(), 1,
                   n_z, w, ws.data_ptr() if ws is not None else None, nb, N.stream_ptr())
        return tile

    def gather(self, tile, recv=None, group=None, dst: int = 0):
        """THE collective: gather every rank's tile to `dst` (one row each of
        `recv`).  Returns `recv` on dst, None elsewhere."""
        import torch.distributed as dist

        me = dist.get_rank(group)
        dst_g = dist.get_global_rank(group, dst) if group is not None else dst
        dist.gather(tile, gather_list=list(recv.unbind(0)) if me == dst else None, dst=dst_g,
                    group=group)
        return recv if me == dst else None

    def display(self, recv, range_db: float, out=None):
        """Display [n_z, n_x] of the gathered tiles (bm_display_tiles, on the
        destination's device).  Returns (display, status)."""
        import torch

        from . import _native as N

        n_z, n_x = self.grid.n_z, self.grid.n_x
        code = N.BM_F32 if recv.dtype == torch.float32 else N.BM_F64
        if out is None:
            out = torch.empty((n_z, n_x), dtype=recv.dtype, device=recv.device)
        status = torch.empty(1, dtype=torch.int32, device=recv.device)
        with torch.cuda.device(recv.device):
            N.call("bm_display_tiles", code, recv.data_ptr(), self.world, self.tile_stride, n_z,
                   n_x, out.data_ptr(), status.data_ptr(), float(range_db), N.stream_ptr())
        return out, status


class PeerTiles:
    """The column split's gather done by the envelope kernel itself, over
    NVLink peer memory (torch symmetric memory maps every rank's receive
    buffer into every process):

      rank r:   wait until its slot is free (device-side flag)
                bm_envelope_peak writes the slab's envelope AND its peak
                  straight into the destination's receive row r (peer stores
                  and a peer atomicMax -- the transfer IS the kernel's output)
                raise ready[r] on the destination (system-scope release)
      dst:      wait for every ready[r] (device-side acquire)
                bm_display_tiles over the rows, then free every rank's slot

    No collective kernel and no host synchronisation: frames are ordered by
    per-rank epoch flags, so the DAS of frame e + 1 overlaps the transfer and
    display of frame e.  Same tile layout and kernels as LateralSplit's NCCL
    gather, so the display is the same bits."""

    def __init__(self, split: "LateralSplit", device, group=None, dst: int = 0):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        self.split, self.dst, self.device = split, int(dst), device
        world, me = split.world, split.rank
        g = group if group is not None else dist.group.WORLD
        self.recv = symm.empty((world, split.tile_stride), dtype=torch.float32, device=device)
        # flags[0][r]: tile r ready (on dst); flags[1][0]: this rank's slot free
        self.flags = symm.empty((2, world), dtype=torch.int32, device=device)
        self.flags.zero_()
        torch.cuda.synchronize(device)
        self.h_recv = symm.rendezvous(self.recv, g)
        self.h_flags = symm.rendezvous(self.flags, g)
        dist.barrier(g)
        self.tile_ptr = self.h_recv.buffer_ptrs[self.dst] + me * split.tile_stride * 4
        self.ready_ptr = self.h_flags.buffer_ptrs[self.dst] + me * 4
        self.free_ptrs = [p + world * 4 for p in self.h_flags.buffer_ptrs]
        self.is_dst = me == self.dst
        self.epoch = 0
        self._ws = None

    def step(self, rf_slab, range_db: float, out=None):
        """One frame: this rank's slab [n_z, w] -> its tile on dst; returns
        (display, status) on dst, None elsewhere.  Enqueued on the current
        stream."""
        import torch

        from . import _native as N

        sp = self.split
        self.epoch += 1
        e = self.epoch
        n_z, w = rf_slab.shape
        x = rf_slab.contiguous()
        s = N.stream_ptr()
        with torch.cuda.device(self.device):
            lib = N.load()
            N.call("bm_wait_flags", self.flags.data_ptr() + sp.world * 4, 1, e - 1, s)
            nb = int(lib.bm_sigproc_ws_bytes(N.SIG_ENVELOPE_PEAK, N.BM_F32, 1, n_z, w))
            if nb and (self._ws is None or self._ws.numel() < nb):
                self._ws = N.workspace(nb, self.device)
            N.call("bm_envelope_peak", N.BM_F32, x.data_ptr(), self.tile_ptr,
                   self.tile_ptr + (sp.tile_stride - 1) * 4, 1, n_z, w,
                   self._ws.data_ptr() if nb else None, nb, s)
            N.call("bm_signal_flag", self.ready_ptr, e, s)
            if not self.is_dst:
                return None
            N.call("bm_wait_flags", self.flags.data_ptr(), sp.world, e, s)
            disp, status = sp.display(self.recv, range_db, out=out)
            for p in self.free_ptrs:
                N.call("bm_signal_flag", p, e, s)
        return disp, status


def row_bands(n_z: int, world: int) -> list[tuple[int, int]]:
    """[lo, hi) depth-row ranges, one per rank, sizes differing by <= 1."""
    return column_slabs(n_z, world)


class RowSplit:
    """Depth-band decomposition of one frame's image grid."""

    def __init__(self, grid, world: int, rank: int):
        self.grid, self.world, self.rank = grid, int(world), int(rank)
        self.bands = row_bands(grid.n_z, self.world)
        lo, hi = self.bands[self.rank]
        if hi <= lo:
            raise ValueError(f"rank {rank} has no rows ({grid.n_z} rows, {world} ranks)")
        self.lo, self.hi = lo, hi
        self.sub_grid = ImageGrid(np.asarray(grid.x_positions),
                                  np.asarray(grid.z_positions)[lo:hi])

    @property
    def band_rows(self) -> int:
        return max(b - a for a, b in self.bands)

    def send_band(self, dtype, device):
        """[band_rows, n_x] send buffer; DAS writes this rank's rows into its top."""
        import torch

        return torch.zeros((self.band_rows, self.grid.n_x), dtype=dtype, device=device)

    def recv_bands(self, dtype, device):
        import torch

        return torch.zeros((self.world, self.band_rows, self.grid.n_x), dtype=dtype,
                           device=device)

    def gather(self, band, recv=None, group=None, dst: int = 0):
        """Gather every rank's band to `dst`; returns the stitched frame
        [n_z, n_x] there (a view when the bands are equal, else one copy),
        None elsewhere."""
        import torch
        import torch.distributed as dist

        me = dist.get_rank(group)
        dst_g = dist.get_global_rank(group, dst) if group is not None else dst
        dist.gather(band, gather_list=list(recv.unbind(0)) if me == dst else None, dst=dst_g,
                    group=group)
        if me != dst:
            return None
        h = self.band_rows
        if all(b - a == h for a, b in self.bands):
            return recv.view(self.world * h, self.grid.n_x)
        return torch.cat([recv[r, : b - a] for r, (a, b) in enumerate(self.bands)], dim=0)


class PeerBands:
    """The depth-row split's gather done by the DAS kernel itself: rank 0's
    frame buffer is symmetric memory mapped into every rank, and each rank's
    bm_das_beamform stores its band's rows straight into it (NVLink peer
    stores); flags as in PeerTiles, then rank 0 runs the fused envelope +
    display of the whole frame."""

    def __init__(self, split: "RowSplit", device, group=None, dst: int = 0):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm

        self.split, self.dst, self.device = split, int(dst), device
        world, me = split.world, split.rank
        g = group if group is not None else dist.group.WORLD
        n_z, n_x = split.grid.n_z, split.grid.n_x
        self.frame = symm.empty((n_z, n_x), dtype=torch.float32, device=device)
        self.flags = symm.empty((2, world), dtype=torch.int32, device=device)
        self.flags.zero_()
        torch.cuda.synchronize(device)
        self.h_frame = symm.rendezvous(self.frame, g)
        self.h_flags = symm.rendezvous(self.flags, g)
        dist.barrier(g)
        # this rank's rows of the destination's frame, as a tensor the DAS
        # launch writes (a peer mapping of the destination's memory)
        self.band = self.h_frame.get_buffer(self.dst, (split.hi - split.lo, n_x), torch.float32,
                                            split.lo * n_x)
        self.ready_ptr = self.h_flags.buffer_ptrs[self.dst] + me * 4
        self.free_ptrs = [p + world * 4 for p in self.h_flags.buffer_ptrs]
        self.is_dst = me == self.dst
        self.epoch = 0

    def step(self, plan, rf, range_db: float):
        """One frame: DAS of this rank's band into the destination's frame;
        returns (display, status) on dst, None elsewhere."""
        import torch

        from . import _native as N

        self.epoch += 1
        e = self.epoch
        s = N.stream_ptr()
        with torch.cuda.device(self.device):
            N.call("bm_wait_flags", self.flags.data_ptr() + self.split.world * 4, 1, e - 1, s)
            plan.beamform_batch(rf, out=self.band[None])
            N.call("bm_signal_flag", self.ready_ptr, e, s)
            if not self.is_dst:
                return None
            N.call("bm_wait_flags", self.flags.data_ptr(), self.split.world, e, s)
            res = envelope_display(self.frame, range_db)
            for p in self.free_ptrs:
                N.call("bm_signal_flag", p, e, s)
        return res


def envelope_display(rf_img, range_db: float):
    """Envelope + dB display of one beamformed frame [n_z, n_x] on its device
    (the fused bm_envelope_display of the single-GPU chain).  Returns
    (display, status)."""
    import torch

    from . import _native as N

    x = rf_img.contiguous()
    code = N.BM_F32 if x.dtype == torch.float32 else N.BM_F64
    peak = torch.empty(1, dtype=_peak_dtype(x.dtype), device=x.device)
    disp = torch.empty_like(x)
    status = torch.empty(1, dtype=torch.int32, device=x.device)
    n_z, n_x = x.shape
    with torch.cuda.device(x.device):
        nb = int(N.load().bm_sigproc_ws_bytes(N.SIG_ENVELOPE_DISPLAY, code, 1, n_z, n_x))
        ws = N.workspace(nb, x.device)
        N.call("bm_envelope_display", code, x.data_ptr(), disp.data_ptr(), peak.data_ptr(),
               status.data_ptr(), 1, n_z, n_x, float(range_db), ws.data_ptr(), nb,
               N.stream_ptr())
    return disp, status
