"""GPU: the per-rank compute of the multi-GPU splits of one large frame
(config 5) on one device.  Ranks are run one after another (no collective:
ranks whose kernels wait on each other must not share a GPU); the tiles /
bands they would send are stacked as the gather delivers them, and dst's
display must equal the single-frame run bitwise (DAS per pixel, FFT per
column, the same display mapping with the same global peak)."""

import numpy as np
import pytest

import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import environment as ME
from paper_1811_01566_b200 import parallel as P

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n_z,n_x,world", [(256, 200, 3), (2048, 96, 2), (300, 61, 4),
                                            (512, 256, 8)])
def test_lateral_tiles_equal_full_frame(n_z, n_x, world):
    import torch

    ctx, grid, n_s = ME.config_geometry("cfg5", n_z=n_z, n_x=n_x)
    rf = torch.from_numpy(np.random.default_rng(5).normal(size=(128, 128, n_s))
                          .astype(np.float32)).cuda()
    full = bm.BmodeEngine(ctx, grid)
    disp_full = full.reconstruct(rf[None])[0].clone()
    rf_full = full._buffers(1)[1][0].clone()
    split0 = P.LateralSplit(grid, world, 0)
    recv = split0.recv_tiles(torch.float32, "cuda")
    rf_parts = []
    for r in range(world):
        split = P.LateralSplit(grid, world, r)
        eng = bm.BmodeEngine(ctx, split.sub_grid)
        slab = eng.plan.beamform_batch(rf[None])[0]
        rf_parts.append(slab.clone())
        split.envelope_into_tile(slab, recv[r])  # rank r's send tile, as gathered
    assert torch.equal(torch.cat(rf_parts, 1), rf_full)
    disp, status = split0.display(recv, 30.0)
    assert int(status.item()) == 0
    if all(lo % 2 == 0 for lo, _ in split0.slabs):
        # K2 packs column pairs (2c, 2c + 1) into one complex transform: slabs
        # starting on even columns pair them as the full frame does -- bitwise
        assert torch.equal(disp, disp_full)
    else:  # other pairings differ by FFT round-off only
        assert float((disp - disp_full).abs().max()) <= 2e-5
        assert float(disp.max()) == 1.0


def test_lateral_tiles_all_zero_frame_sets_status():
    import torch

    ctx, grid, n_s = ME.config_geometry("cfg5", n_z=64, n_x=40)
    world = 2
    recv = P.LateralSplit(grid, world, 0).recv_tiles(torch.float32, "cuda")
    for r in range(world):
        split = P.LateralSplit(grid, world, r)
        split.envelope_into_tile(torch.zeros((64, split.hi - split.lo), device="cuda"), recv[r])
    disp, status = P.LateralSplit(grid, world, 0).display(recv, 30.0)
    assert int(status.item()) == 1 and float(disp.abs().max()) == 0.0


def test_row_bands_equal_full_frame():
    """Depth bands of config 5's split by rows, beamformed one after another on
    one device and stacked: rf bitwise the full frame's; the destination's
    envelope + display of the stacked frame bitwise the single-GPU chain."""
    import torch

    ctx, grid, n_s = ME.config_geometry("cfg5", n_z=200, n_x=96)
    rf = torch.from_numpy(np.random.default_rng(6).normal(size=(128, 128, n_s))
                          .astype(np.float32)).cuda()
    full = bm.BmodeEngine(ctx, grid)
    disp_full = full.reconstruct(rf[None])[0].clone()
    rf_full = full._buffers(1)[1][0].clone()
    world = 3
    split0 = P.RowSplit(grid, world, 0)
    recv = split0.recv_bands(torch.float32, "cuda")
    for r in range(world):
        split = P.RowSplit(grid, world, r)
        eng = bm.BmodeEngine(ctx, split.sub_grid)
        eng.plan.beamform_batch(rf[None], out=recv[r, None, : split.hi - split.lo])
    stacked = torch.cat([recv[r, : b - a] for r, (a, b) in enumerate(split0.bands)], 0)
    assert torch.equal(stacked, rf_full)
    disp, status = P.envelope_display(stacked, 30.0)
    assert int(status.item()) == 0
    assert torch.equal(disp, disp_full)


def test_peer_tiles_envelope_kernel_writes_the_gather():
    """The NVLink peer-memory form of the column split (parallel.PeerTiles):
    bm_envelope_peak writes each rank's [envelope | peak] tile straight into
    the destination's symmetric receive buffer, device-side epoch flags order
    the frames, and the destination's display equals the one-GPU chain bitwise
    -- over several back-to-back frames with no host synchronisation between
    them.  One rank here (the peer mapping is the rank's own buffer): ranks
    whose kernels wait on each other must not share a GPU."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        ctx, grid, n_s = ME.config_geometry("cfg5", n_z=256, n_x=200)
        split = P.LateralSplit(grid, 1, 0)
        peer = P.PeerTiles(split, torch.device("cuda", 0))
        full = bm.BmodeEngine(ctx, grid)
        g = torch.Generator(device="cuda").manual_seed(9)
        frames = [torch.randn((1, 128, 128, n_s), generator=g, device="cuda") for _ in range(3)]
        outs = []
        for rf in frames:
            slab = full.plan.beamform_batch(rf)[0]
            disp, status = peer.step(slab, 30.0)
            outs.append((disp.clone(), status.clone()))
        for rf, (disp, status) in zip(frames, outs):
            assert int(status.item()) == 0
            assert torch.equal(disp, full.reconstruct(rf)[0])
        assert peer.epoch == 3
        # the depth-row split: the DAS kernel stores its band into the
        # destination's frame buffer
        rsplit = P.RowSplit(grid, 1, 0)
        bands = P.PeerBands(rsplit, torch.device("cuda", 0))
        outs = [tuple(t.clone() for t in bands.step(full.plan, rf, 30.0)) for rf in frames]
        for rf, (disp, status) in zip(frames, outs):
            assert int(status.item()) == 0
            assert torch.equal(disp, full.reconstruct(rf)[0])
    finally:
        dist.destroy_process_group()
