"""Parity of the path bench.py times: ``BmodeEngine.reconstruct`` on the
bench's own cine batches (bench.synth_frames) against outputs of the
reference (tests/golden/engine.npz, written by make_golden.py running
echopipe on the same frames).

Per golden frame of the batch:
  * the f32 input RF is byte-identical to the reference's input (sha256);
  * the beamformed RF (DAS output, the engine's rf workspace) is bitwise the
    reference's das_beamform output (sha256);
  * the display is within 2e-5 (abs, display in [0, 1]) of the reference
    chain's (FFT round-off differs from pocketfft; argmax and zeros exact).

The launch shape is asserted, so the multi-frame passes (FP warp groups x FT
frames per thread) are what is being checked.
"""

import hashlib
import os

import numpy as np
import pytest

import bench
import cases
import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import environment as ME

pytestmark = pytest.mark.gpu

DISP_TOL = 2e-5


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def eg(golden_dir):
    return np.load(os.path.join(golden_dir, "engine.npz"))


def _golden_seeds(eg, name, kind):
    pre = f"{name}_{kind}_"
    return sorted(int(k[len(pre):]) for k in eg.files if k.startswith(pre))


def _check_batch(eg, name, n_frames, fp, ft):
    import torch

    ctx, grid, n_s = ME.config_geometry(name)
    host = bench.synth_frames(ctx, n_s, n_frames, 0)
    for s in _golden_seeds(eg, name, "in_sha"):
        assert sha(host[s]) == str(eg[f"{name}_in_sha_{s}"]), f"{name} input frame {s} differs"
    eng = bm.BmodeEngine(ctx, grid)
    shape = eng.plan.launch_shape(n_s, n_frames)
    assert shape is not None and (shape["fp"], shape["ft"]) == (fp, ft), shape
    rf = torch.from_numpy(host).cuda()
    disp = eng.reconstruct(rf)
    torch.cuda.synchronize()
    eng.check()
    rf_img = eng._buffers(n_frames)[1][:n_frames].cpu().numpy()
    disp = disp.cpu().numpy()
    for s in _golden_seeds(eg, name, "rf_sha"):
        assert sha(rf_img[s]) == str(eg[f"{name}_rf_sha_{s}"]), f"{name} frame {s}: DAS not bitwise"
    for s in _golden_seeds(eg, name, "disp"):
        ref = eg[f"{name}_disp_{s}"]
        d = disp[s]
        assert d.dtype == np.float32 and d.shape == ref.shape
        assert float(np.abs(d - ref).max()) <= DISP_TOL, f"{name} frame {s} display"
        assert d.max() == 1.0 and d[ref == 1.0].min() == 1.0
    return eng, host, disp


def test_cfg2_cine_batch_vs_reference(eg):
    """The default bench workload: 32 cfg2 frames, FP = 2 x FT = 4."""
    _check_batch(eg, "cfg2", 32, 2, 4)


def test_cfg1_cine_batch_vs_reference(eg):
    _check_batch(eg, "cfg1", 32, 1, 4)


def test_cfg3_batch_vs_reference(eg):
    _check_batch(eg, "cfg3", 8, 2, 4)


def test_host_stream_equals_device_batch(eg):
    """reconstruct_host_stream (the bench's e2e path: pinned H2D, chunked
    copy/compute overlap, D2H) returns the device path's displays bitwise."""
    import torch

    eng, host, disp = _check_batch(eg, "cfg2", 32, 2, 4)
    rf_h, disp_h = eng.pinned(32, host.shape[-1])
    rf_h.copy_(torch.from_numpy(host))
    eng.reconstruct_host_stream([(rf_h, disp_h), (rf_h, disp_h)], chunk=8)
    eng.check()
    assert np.array_equal(disp_h.numpy(), disp)
    # odd chunking across batch boundaries
    d2 = torch.empty_like(disp_h)
    eng.reconstruct_host_stream([(rf_h[:13], disp_h[:13]), (rf_h[13:], d2[13:])], chunk=5)
    assert np.array_equal(disp_h[:13].numpy(), disp[:13])
    assert np.array_equal(d2[13:].numpy(), disp[13:])


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_engine_on_the_chain_cases(golden_dir, dtype):
    """BmodeEngine (DAS + the fused or two-launch K2/K3) on the six chain
    instances -- STA/PW, rx maps, t0, Hann + F-number, nearest, odd n_z (the
    mixed-radix lane kernel) -- in f32 and f64, as 3-frame batches (the frame,
    the frame x 2, the frame again): the display of every frame equals the
    reference chain's (f32 <= 2e-5, f64 <= 1e-9), the rf image is bitwise."""
    import torch

    from paper_1811_01566_b200 import types as T

    g = np.load(os.path.join(golden_dir, "chain.npz"))
    for name, ctx, data, grid, apod, interp in cases.chain_cases(T):
        dt = np.float32 if dtype == "f32" else np.float64
        x = data.astype(dt)
        batch = torch.from_numpy(np.stack([x, 2 * x, x])).cuda()
        n_rx = data.shape[1]
        eng = bm.BmodeEngine(ctx, grid, apod=apod, interp=interp, dtype=dt, n_rx=n_rx)
        disp = eng.reconstruct(batch).cpu().numpy()
        eng.check()
        rf = eng._buffers(3)[1][:3].cpu().numpy()
        ref_rf = g[f"{name}_rf"] if dtype == "f32" else g[f"{name}_rf64"]
        ref = g[f"{name}_disp"] if dtype == "f32" else g[f"{name}_disp64"]
        tol = 2e-5 if dtype == "f32" else 1e-9
        assert rf[0].tobytes() == ref_rf.tobytes(), name
        for f in range(3):
            assert float(np.abs(disp[f] - ref).max()) <= tol, (name, f)
        assert disp[0].max() == 1.0 and disp[1].max() == 1.0

