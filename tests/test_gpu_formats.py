"""GPU half of the ingest / output formats: write_pgm's pixel quantisation
(bm_quantize_u8) against the reference's bytes (formats.py:189-200,
test_formats.py:107-133, tests/golden/pgm.npz), and WFRF file streaming
through BmodeEngine.reconstruct_file (pinned read_into batches, overlapped
H2D) against the device-resident reconstruction, bitwise."""

import os

import numpy as np
import pytest

import paper_1811_01566_b200 as bm
from paper_1811_01566_b200.errors import WrongStage

pytestmark = pytest.mark.gpu


def grid_1xn(n):
    return bm.ImageGrid(np.arange(n, dtype=np.float64) * 1e-3, np.array([0.0]))


def test_pgm_reference_kats(tmp_path):
    img = bm.BmodeImage(np.array([[1.0]]), stage="display", grid=grid_1xn(1))
    bm.write_pgm(img, tmp_path / "a.pgm")
    assert (tmp_path / "a.pgm").read_bytes() == b"P5\n1 1\n255\n\xff"
    img = bm.BmodeImage(np.array([[0.0, 0.5, 1.0]]), stage="display", grid=grid_1xn(3))
    bm.write_pgm(img, tmp_path / "c.pgm")
    assert (tmp_path / "c.pgm").read_bytes().endswith(bytes([0, 128, 255]))
    with pytest.raises(WrongStage):
        bm.write_pgm(bm.BmodeImage(np.array([[2.0]]), stage="envelope", grid=grid_1xn(1)),
                     tmp_path / "x.pgm")


@pytest.mark.parametrize("name", ["f32", "f64"])
def test_pgm_bytes_equal_reference(golden_dir, tmp_path, name):
    g = np.load(os.path.join(golden_dir, "pgm.npz"))
    d = g[f"disp_{name}"]
    img = bm.BmodeImage(d, stage="display",
                        grid=bm.ImageGrid(np.arange(d.shape[1]) * 1e-4, np.arange(d.shape[0]) * 1e-4))
    path = tmp_path / "g.pgm"
    bm.write_pgm(img, path)
    assert path.read_bytes() == g[f"pgm_{name}"].tobytes()


def test_reconstruct_file_equals_device_reconstruction(tmp_path):
    import torch

    ctx, grid, n_s = bm.environment.config_geometry("cfg2", n_z=96, n_x=80)
    rng = np.random.default_rng(12)
    n = 21  # not a multiple of the batch or the chunk
    rf = rng.normal(size=(n, ctx.n_tx, ctx.n_elements, n_s)).astype(np.float32)
    path = tmp_path / "cine.wfrf"
    bm.write_wfrf(path, [bm.RfFrame(f) for f in rf], ctx)
    eng = bm.BmodeEngine(ctx, grid)
    disp, ctx2 = eng.reconstruct_file(path, batch=8, chunk=3)
    eng.check()
    ref = eng.reconstruct(torch.from_numpy(rf).cuda())
    torch.cuda.synchronize()
    assert disp.shape == (n,) + grid.shape
    assert torch.equal(disp, ref.cpu())
    assert ctx2.n_tx == ctx.n_tx


def test_quantize_vector_and_scalar_paths_equal_numpy():
    """bm_quantize_u8 on f32: the four-pixels-per-thread path (aligned
    buffers), its scalar tail and the unaligned scalar path all equal
    numpy's f32 floor(v * 255 + 0.5), including values on the .5 steps."""
    import torch

    from paper_1811_01566_b200 import _native as N

    rng = np.random.default_rng(3)
    steps = (np.arange(256, dtype=np.float32) + np.float32(0.5)) / np.float32(255)
    for count in (1, 3, 4, 5, 1027, 1 << 16):
        for off in (0, 1, 3):
            v = rng.random(count + off, dtype=np.float32)
            v[off::5] = steps[rng.integers(0, 255, size=len(v[off::5]))]
            v[off::7] = np.nextafter(v[off::7], np.float32(0))
            d = torch.from_numpy(v).cuda()[off:]
            q = torch.empty(count + off, dtype=torch.uint8, device="cuda")[off:]
            N.call("bm_quantize_u8", N.BM_F32, d.data_ptr(), q.data_ptr(), count, N.stream_ptr())
            ref = np.floor(v[off:] * np.float32(255) + np.float32(0.5)).astype(np.uint8)
            assert np.array_equal(q.cpu().numpy(), ref), (count, off)
