"""GPU: the per-rank compute of the lateral split (config 5) on one device.
Slabs are reconstructed one after another (no collective -- ranks whose
kernels wait on each other must not share a GPU); stitched, they must equal
the single-frame run: rf bitwise, envelope bitwise (same per-column FFT),
display identical once mapped with the global peak."""

import numpy as np
import pytest

import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import environment as ME
from paper_1811_01566_b200 import parallel as P

pytestmark = pytest.mark.gpu


def test_lateral_slabs_equal_full_frame():
    import torch

    ctx, grid, n_s = ME.config_geometry("cfg5", n_z=256, n_x=200)
    rf = torch.from_numpy(np.random.default_rng(5).normal(size=(128, 128, n_s))
                          .astype(np.float32)).cuda()
    full = bm.BmodeEngine(ctx, grid)
    disp_full = full.reconstruct(rf[None])[0]
    rf_full = full._buffers(1)[1][0].clone()
    env_full = full._buffers(1)[2][0].clone()
    world = 3
    rf_parts, env_parts, peaks = [], [], []
    for r in range(world):
        split = P.LateralSplit(grid, world, r)
        eng = bm.BmodeEngine(ctx, split.sub_grid)
        eng.reconstruct(rf[None])
        rf_parts.append(eng._buffers(1)[1][0].clone())
        env_parts.append(eng._buffers(1)[2][0].clone())
        peaks.append(float(env_parts[-1].max()))
    assert torch.equal(torch.cat(rf_parts, 1), rf_full)
    assert torch.equal(torch.cat(env_parts, 1), env_full)
    gpeak = max(peaks)
    disp = torch.cat([P.map_display(e, gpeak, 30.0) for e in env_parts], 1)
    assert torch.equal(disp, disp_full)


def test_row_bands_equal_full_frame():
    """Depth bands of config 5's split by rows, beamformed one after another on
    one device and stacked: rf bitwise the full frame's; the destination's
    envelope + display of the stacked frame bitwise the single-GPU chain."""
    import torch

    ctx, grid, n_s = ME.config_geometry("cfg5", n_z=200, n_x=96)
    rf = torch.from_numpy(np.random.default_rng(6).normal(size=(128, 128, n_s))
                          .astype(np.float32)).cuda()
    full = bm.BmodeEngine(ctx, grid)
    disp_full = full.reconstruct(rf[None])[0]
    rf_full = full._buffers(1)[1][0].clone()
    world = 3
    bands = []
    for r in range(world):
        split = P.RowSplit(grid, world, r)
        eng = bm.BmodeEngine(ctx, split.sub_grid)
        eng.reconstruct(rf[None])
        bands.append(eng._buffers(1)[1][0].clone())
    stacked = torch.cat(bands, 0)
    assert torch.equal(stacked, rf_full)
    disp, _ = P.envelope_display(stacked, 30.0)
    assert torch.equal(disp, disp_full)
