"""GPU parity of the RF pre-filter:
sigproc.fir_filter (sigproc.py:36-45) and the `fir_filter` operator
(pipeline.py:96-105) against the reference's outputs (tests/golden/fir.npz,
made by running echopipe) and its own KATs (test_sigproc.py:19-61,
test_acceptance.py:190-195, test_pipeline.py:205-216).

Tolerances: the reference sums each output with numpy's BLAS dot (an
implementation-defined order); the kernel sums oldest tap first in f64.
  f64 results:           max|dy| <= 1e-13 * sum_m |h[m]| * max|x|
  f32 frames (operator): the f64 result rounded once to f32, so equal to the
                         reference's cast up to one f32 ulp.
"""

import os

import numpy as np
import pytest

import paper_1811_01566_b200 as bm
from paper_1811_01566_b200.errors import AxisTooShort, EmptyCoefficients

pytestmark = pytest.mark.gpu

NT = (1, 2, 7, 33, 64)


@pytest.fixture(scope="module")
def g(golden_dir):
    return np.load(os.path.join(golden_dir, "fir.npz"))


@pytest.mark.parametrize("nt", NT)
def test_fir_vs_reference_goldens(g, nt):
    h = g[f"h_{nt}"]
    spec = bm.FirSpec(h)
    for xk, yk, ax in (("x32", "y32", -1), ("x64", "y64", -1), ("xa", "ya", 0)):
        x, ref = g[f"{xk}_{nt}"], g[f"{yk}_{nt}"]
        y = bm.fir_filter(x, spec, axis=ax)
        assert y.dtype == np.float64 and y.shape == ref.shape
        bound = 1e-13 * np.abs(h).sum() * np.abs(x).max()
        assert np.abs(y - ref).max() <= bound, (nt, xk, np.abs(y - ref).max())


@pytest.mark.parametrize("nt", NT)
def test_fir_operator_keeps_frame_dtype(g, nt):
    """The operator returns a frame of the input dtype: the f64 result
    rounded once (pipeline.py:104)."""
    import torch

    op = bm.OPERATOR_REGISTRY["fir_filter"].factory({"coefficients": list(g[f"h_{nt}"])})
    x = g[f"x32_{nt}"]
    frame, ctx = op((bm.RfFrame(x), "ctx"))
    assert ctx == "ctx"
    y = frame.data
    assert isinstance(y, torch.Tensor) and y.dtype == torch.float32 and y.is_cuda
    y = y.cpu().numpy()
    ref = g[f"y32_{nt}"].astype(np.float32)
    assert np.all(np.abs(y - ref) <= np.spacing(np.abs(ref)))
    assert np.mean(y == ref) > 0.999


def test_fir_impulse_response_equals_coefficients():
    y = bm.fir_filter(np.array([1.0, 0.0, 0.0, 0.0]), bm.FirSpec([0.5, 0.5]))
    np.testing.assert_array_equal(y, [0.5, 0.5, 0.0, 0.0])


def test_fir_identity():
    x = np.random.default_rng(0).normal(size=(3, 17))
    np.testing.assert_array_equal(bm.fir_filter(x, bm.FirSpec([1.0])), x)


def test_fir_hand_convolution():
    y = bm.fir_filter(np.array([1.0, 2.0, 3.0]), bm.FirSpec([1.0, 1.0]))
    np.testing.assert_allclose(y, [1.0, 3.0, 5.0])


def test_fir_along_chosen_axis():
    x = np.zeros((4, 3))
    x[0] = 1.0
    y = bm.fir_filter(x, bm.FirSpec([1.0, -1.0]), axis=0)
    np.testing.assert_allclose(y[0], 1.0)
    np.testing.assert_allclose(y[1], -1.0)
    np.testing.assert_allclose(y[2:], 0.0)


def test_fir_linearity_and_shift():
    rng = np.random.default_rng(3)
    spec = bm.FirSpec(rng.normal(size=5))
    x1, x2 = rng.normal(size=64), rng.normal(size=64)
    np.testing.assert_allclose(bm.fir_filter(x1 + 2.0 * x2, spec),
                               bm.fir_filter(x1, spec) + 2.0 * bm.fir_filter(x2, spec),
                               rtol=1e-12)
    shifted = np.concatenate([[0.0], x1[:-1]])
    np.testing.assert_allclose(bm.fir_filter(shifted, spec)[1:], bm.fir_filter(x1, spec)[:-1])


def test_fir_acceptance_impulse():
    taps = np.array([0.25, -0.5, 1.0, 0.125])
    impulse = np.zeros(16)
    impulse[0] = 1.0
    response = bm.fir_filter(impulse, bm.FirSpec(taps))
    np.testing.assert_array_equal(response[:4], taps)
    np.testing.assert_array_equal(response[4:], 0.0)


def test_fir_errors():
    with pytest.raises(EmptyCoefficients):
        bm.FirSpec([])
    with pytest.raises(EmptyCoefficients):
        bm.FirSpec([1.0, np.nan])
    with pytest.raises(AxisTooShort):
        bm.fir_filter(np.zeros((3, 0)), bm.FirSpec([1.0]))


def test_fir_long_filter_and_device_tensors():
    """Taps longer than a 256-sample tile, device tensor in -> device tensor out."""
    import torch

    rng = np.random.default_rng(5)
    h = rng.normal(size=300)
    x = rng.normal(size=(4, 1000)).astype(np.float32)
    ref = np.stack([np.convolve(h, r.astype(np.float64))[:1000] for r in x])
    y = bm.fir_filter(torch.from_numpy(x).cuda(), bm.FirSpec(h))
    assert y.is_cuda and y.dtype == torch.float64
    assert np.abs(y.cpu().numpy() - ref).max() <= 1e-13 * np.abs(h).sum() * np.abs(x).max()


def test_fir_node_prefilters_frame():
    spec = bm.bmode_chain()
    spec["nodes"].append(
        {"name": "fir", "kind": "fir_filter", "params": {"coefficients": [0.5, 0.5]}})
    spec["edges"].insert(0, {"from": "fir", "to": "beamform"})
    spec["inputs"] = ["fir"]
    graph = bm.build_graph(spec)
    ctx, grid, n_s = bm.environment.config_geometry("cfg1", n_z=64, n_x=64, n_tx=8)
    rng = np.random.default_rng(1)
    frame = bm.RfFrame(rng.normal(size=(ctx.n_tx, ctx.n_elements, n_s)).astype(np.float32))
    outputs, timing = bm.execute(graph, (frame, ctx))
    assert outputs["dynamic_adjustment"].stage == "display"
    assert [s for s, _ in timing.stages][0] == "fir"


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("M", [1, 5, 64, 300, 1500])
def test_fir_row_kernel_bitwise_equals_one_output_kernel(dtype, M, monkeypatch):
    """Contiguous lanes run the register-blocked kernel (four outputs per
    thread); it must equal the one-output kernel bit for bit, lengths not a
    multiple of its 1024-output tile, shorter than the filter, and -0.0
    products against the zero initial state included."""
    import torch

    rng = np.random.default_rng(M)
    h = rng.normal(size=M)
    h[0] = -abs(h[0])  # a negative newest tap: h*0 = -0.0 at a zero sample
    for n in (1, 3, 1023, 1025, 2048 + 77):
        x = rng.normal(size=(5, n)).astype(dtype)
        x[:, ::7] = 0.0
        xd = torch.from_numpy(x).cuda()
        blocked = bm.fir_filter(xd, bm.FirSpec(h)).cpu().numpy()
        monkeypatch.setenv("BM_FIR_ONE_OUTPUT", "1")
        one = bm.fir_filter(xd, bm.FirSpec(h)).cpu().numpy()
        monkeypatch.delenv("BM_FIR_ONE_OUTPUT")
        assert blocked.tobytes() == one.tobytes(), (M, n)
