"""Multi-process (gloo, world_size 2, CPU) tests of the multi-GPU logic:
frame partitioning, the lateral column split of one large frame (one gather
of [envelope | peak] tiles to the destination) and the depth-row split (one
gather of RF bands).  Per-rank
compute is the CPU oracle here (test infrastructure); on GPUs it is the
bm_* kernels (tests/test_gpu_parallel.py checks that path on one device)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1811_01566_b200 import parallel as P
from paper_1811_01566_b200 import types as T


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_frame_partition_covers_all_frames():
    for n in (0, 1, 7, 256):
        for world in (1, 2, 3, 8):
            got = [i for r in range(world) for i in P.frame_partition(n, world, r)]
            assert got == list(range(n))
            sizes = [len(P.frame_partition(n, world, r)) for r in range(world)]
            assert max(sizes) - min(sizes) <= 1


def test_column_slabs():
    assert P.column_slabs(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert P.column_slabs(2048, 8)[7] == (1792, 2048)


def _geometry():
    ctx = T.AcquisitionContext(1540.0, 40e6, 16, 2e-4, T.StaScheme(tuple(range(16))))
    ex = ctx.element_positions()
    grid = T.ImageGrid(np.linspace(ex[0], ex[-1], 37), np.linspace(0, 512 * 1540 / 80e6, 64))
    rf = np.random.default_rng(3).normal(size=(16, 16, 512)).astype(np.float32)
    return ctx, grid, rf


def _worker(rank, world, port, out_path):
    from oracle import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx, grid, rf = _geometry()
        split = P.LateralSplit(grid, world, rank)
        rf_slab = O.das_beamform(rf, ctx, split.sub_grid)                 # per-rank DAS
        env = np.abs(O.analytic_signal(rf_slab, axis=0)).astype(np.float32)  # rank-local lanes
        # the tile bm_envelope_peak fills on a GPU: envelope, then the peak bits
        tile = split.send_tile(torch.float32, "cpu")
        env_v, peak_v = split.tile_views(tile)
        env_v.copy_(torch.from_numpy(env))
        peak_v.copy_(torch.from_numpy(np.array([env.max()], np.float32).view(np.int32)))
        recv = split.recv_tiles(torch.float32, "cpu") if rank == 0 else None
        got = split.gather(tile, recv)                                    # THE collective
        if rank == 0:
            envs = [split.envelope_view(got[r], r).numpy() for r in range(world)]
            peaks = got[:, -1].view(torch.int32).numpy().view(np.float32)
            np.savez(out_path, env=np.concatenate(envs, axis=1), peaks=peaks,
                     widths=np.array([e.shape[1] for e in envs]))
        else:
            assert got is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_lateral_split_gloo_matches_single_process(tmp_path, world):
    """Column split of one frame (cfg5): every rank's [envelope | peak] tile
    reaches dst in one gather, laid out as bm_display_tiles reads it; the
    stitched envelope is the single-process one and the max of the tile peaks
    is its peak, so dst's display is the single-process display."""
    from oracle import oracle as O

    out = str(tmp_path / "out.npz")
    mp.spawn(_worker, args=(world, free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    ctx, grid, rf = _geometry()
    rf_ref, env_ref, disp_ref = O.bmode_chain(rf, ctx, grid)
    assert [h - l for l, h in P.column_slabs(grid.n_x, world)] == list(got["widths"])
    assert np.abs(got["env"] - env_ref).max() <= 1e-6 * env_ref.max()
    assert got["peaks"].max() == got["env"].max()
    # the mapping bm_display_tiles applies, with the gathered global peak
    disp = O.dynamic_adjustment_with_peak(got["env"], got["peaks"].max(), 30.0)
    assert np.abs(disp - disp_ref).max() <= 1e-5
    assert disp.max() == 1.0


def _row_worker(rank, world, port, out_path):
    from oracle import oracle as O

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ctx, grid, rf = _geometry()
        split = P.RowSplit(grid, world, rank)
        send = split.send_band(torch.float32, "cpu")
        band = O.das_beamform(rf, ctx, split.sub_grid)          # per-rank DAS of a depth band
        send[: band.shape[0]] = torch.from_numpy(band)
        recv = split.recv_bands(torch.float32, "cpu") if rank == 0 else None
        rf_full = split.gather(send, recv)                      # the only collective
        if rank == 0:
            np.savez(out_path, rf=rf_full.numpy())
        else:
            assert rf_full is None
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_split_gloo_matches_single_process(tmp_path, world):
    """Depth-band split (RowSplit): the gathered bands are bitwise the
    single-process beamformed frame, so the destination's envelope + display
    of it equal the single-GPU chain."""
    from oracle import oracle as O

    out = str(tmp_path / "rows.npz")
    mp.spawn(_row_worker, args=(world, free_port(), out), nprocs=world, join=True)
    got = np.load(out)
    ctx, grid, rf = _geometry()
    rf_ref, _, _ = O.bmode_chain(rf, ctx, grid)
    assert got["rf"].tobytes() == rf_ref.tobytes()


def test_row_bands():
    assert P.row_bands(10, 3) == [(0, 4), (4, 7), (7, 10)]
    ctx, grid, _ = _geometry()
    bands = [P.RowSplit(grid, 3, r).sub_grid for r in range(3)]
    assert sum(b.n_z for b in bands) == grid.n_z
    assert np.array_equal(np.concatenate([b.z_positions for b in bands]), grid.z_positions)
