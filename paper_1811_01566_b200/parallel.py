"""Multi-GPU partitioning of the B-mode path.

Two cases, one process per GPU (torch.distributed, NCCL on GPUs, gloo in
the CPU tests):

* **Independent frames** (config 4, cine streams): `frame_partition` deals
  frames to ranks; there is no data-path collective.

* **One large frame** (config 5, 2048 x 2048 STAI): `LateralSplit` gives
  every rank a contiguous slab of image COLUMNS at all depths.  Delay-and-
  Sum is per pixel, so each rank's slab is bitwise equal to the same columns
  of a single-GPU run; the analytic signal runs along depth, so every FFT
  lane is rank-local.  The only coupling is the per-frame peak of
  dynamic_adjustment (sigproc.py:90): one all-reduce(MAX) of a single
  float, then each rank maps its slab to display values and one gather
  assembles the B-mode image on the destination rank.

* **One large frame, split by depth ROWS** (`RowSplit`, the north star's
  literal "image rows are split across GPUs"): each rank beamforms a band of
  rows at all columns -- again bitwise the same pixels as one GPU -- but a
  band cuts every axial FFT lane, so the beamformed RF bands are gathered
  to the destination rank, which runs the envelope + display of the whole
  frame (the same kernels as one GPU, so the same bits).  One all-gather of
  f32 RF rows, no other collective.

The per-rank compute is injectable (`local_fn(sub_grid, rank) -> envelope
slab`) so the partition/collective logic is testable on CPU with gloo.
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
    """[lo, hi) column ranges, one per rank, sizes differing by <= 1."""
    return [(r.start, r.stop) for r in (frame_partition(n_x, world, k) for k in range(world))]


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

    def pad_width(self) -> int:
        return max(h - l for l, h in self.slabs)

    def display(self, env_slab, range_db: float, group=None, dst: int = 0):
        """Global-peak dB mapping of this rank's envelope slab, gathered to
        `dst`.  `env_slab` is a torch tensor [n_z, n_cols] (CUDA with NCCL,
        CPU with gloo).  Returns the full [n_z, n_x] display on `dst`, None
        elsewhere."""
        import torch
        import torch.distributed as dist

        peak = env_slab.max().reshape(1).to(torch.float64)
        dist.all_reduce(peak, op=dist.ReduceOp.MAX, group=group)
        disp = map_display(env_slab, float(peak.item()), range_db)
        return self.gather(disp, group=group, dst=dst)

    def gather(self, slab, group=None, dst: int = 0):
        """Gather equal-padded column slabs to `dst` and stitch them."""
        import torch
        import torch.distributed as dist

        n_z = slab.shape[0]
        w = self.pad_width()
        buf = torch.zeros((n_z, w), dtype=slab.dtype, device=slab.device)
        buf[:, : slab.shape[1]] = slab
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf.contiguous(), group=group)
        if dist.get_rank(group) != dst:
            return None
        return torch.cat([p[:, : h - l] for p, (l, h) in zip(parts, self.slabs)], dim=1)


def map_display(env, peak: float, range_db: float):
    """dB mapping of an envelope slab against a GLOBAL peak, on the device
    that holds it: the bm_display kernel for CUDA tensors (same arithmetic as
    the single-GPU path), torch ops for CPU tensors (gloo tests only)."""
    import torch

    if env.is_cuda:
        from . import _native as N

        code = N.BM_F32 if env.dtype == torch.float32 else N.BM_F64
        bits = torch.tensor([peak], dtype=env.dtype).view(
            torch.int32 if code == N.BM_F32 else torch.int64).to(env.device)
        out = torch.empty_like(env)
        status = torch.empty(1, dtype=torch.int32, device=env.device)
        e = env.contiguous()
        N.call("bm_display", code, e.data_ptr(), bits.data_ptr(), out.data_ptr(),
               status.data_ptr(), 1, e.numel(), float(range_db), N.stream_ptr())
        return out
    e = env
    pos = e > 0
    out = torch.zeros_like(e)
    db = 20.0 * torch.log10(e[pos] / e.new_tensor(peak))
    out[pos] = torch.clamp(db + range_db, 0.0, range_db) / range_db
    return out


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

    def gather(self, band, group=None, dst: int = 0):
        """Gather equal-padded row bands [rows, n_x] to `dst` and stack them."""
        import torch
        import torch.distributed as dist

        h = max(b - a for a, b in self.bands)
        buf = torch.zeros((h,) + tuple(band.shape[1:]), dtype=band.dtype, device=band.device)
        buf[: band.shape[0]] = band
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        dist.all_gather(parts, buf.contiguous(), group=group)
        if dist.get_rank(group) != dst:
            return None
        return torch.cat([p[: b - a] for p, (a, b) in zip(parts, self.bands)], dim=0)


def envelope_display(rf_img, range_db: float):
    """Envelope + dB display of one beamformed frame [n_z, n_x] on its device
    (the bm_envelope_peak + bm_display kernels of the single-GPU chain).
    Returns (display, envelope)."""
    import torch

    from . import _native as N

    x = rf_img.contiguous()
    code = N.BM_F32 if x.dtype == torch.float32 else N.BM_F64
    env = torch.empty_like(x)
    peak = torch.empty(1, dtype=torch.int32 if code == N.BM_F32 else torch.int64, device=x.device)
    disp = torch.empty_like(x)
    status = torch.empty(1, dtype=torch.int32, device=x.device)
    n_z, n_x = x.shape
    with torch.cuda.device(x.device):
        N.call("bm_envelope_peak", code, x.data_ptr(), env.data_ptr(), peak.data_ptr(), 1, n_z, n_x,
               N.stream_ptr())
        N.call("bm_display", code, env.data_ptr(), peak.data_ptr(), disp.data_ptr(),
               status.data_ptr(), 1, n_z * n_x, float(range_db), N.stream_ptr())
    return disp, env

