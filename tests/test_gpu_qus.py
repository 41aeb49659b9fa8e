"""GPU parity of the QUS hooks: sliding_moments and
the dense homodyned-K estimator against the reference's outputs
(tests/golden/qus.npz, made by running echopipe) and its own KATs
(test_qus.py, test_acceptance.py:235-247 criterion 7, test_pipeline.py:219-233).

Tolerances: numpy sums windows pairwise and takes x**3 through pow(); the
kernel uses compensated f64 sums and x*x*x, the dense layers sum in lane
order: relative 1e-12 on every map, exact where the reference's KATs are.
"""

import os

import numpy as np
import pytest

import paper_1811_01566_b200 as bm
from paper_1811_01566_b200.errors import DimensionMismatch, InvalidMetadata, WindowTooLarge

pytestmark = pytest.mark.gpu


def one_layer_model():
    return bm.DenseModel((bm.DenseLayer(np.array([[1.0, 1.0, 1.0], [0.0, 0.0, 1.0]]),
                                        np.array([0.0, 1.0]), "identity"),))


def close(a, b, rel=1e-12):
    return np.all(np.abs(a - b) <= rel * np.maximum(np.abs(b), 1e-300))


@pytest.fixture(scope="module")
def g(golden_dir):
    return np.load(os.path.join(golden_dir, "qus.npz"))


@pytest.mark.parametrize("i", range(4))
def test_qus_vs_reference_goldens(g, i):
    img, win, st = g[f"img_{i}"], tuple(g[f"win_{i}"]), tuple(g[f"stride_{i}"])
    maps = bm.sliding_moments(img, win, st)
    for k in ("m1", "m2", "m3"):
        assert getattr(maps, k).shape == g[f"{k}_{i}"].shape
        assert close(getattr(maps, k), g[f"{k}_{i}"]), k
    model = bm.DenseModel(tuple(bm.DenseLayer(g[f"W_{j}"], g[f"b_{j}"], str(a))
                                for j, a in enumerate(g["acts"])))
    hk = bm.estimate_hk_map(img, win, st, model)
    scale = max(np.abs(g[f"u_{i}"]).max(), np.abs(g[f"k_{i}"]).max())
    assert np.abs(hk.u - g[f"u_{i}"]).max() <= 1e-11 * scale
    assert np.abs(hk.k - g[f"k_{i}"]).max() <= 1e-11 * scale


def test_constant_image_moments_exact():
    maps = bm.sliding_moments(np.full((10, 8), 2.0), window=(3, 3), stride=(2, 2))
    np.testing.assert_array_equal(maps.m1, 2.0)
    np.testing.assert_array_equal(maps.m2, 4.0)
    np.testing.assert_array_equal(maps.m3, 8.0)
    assert maps.shape == (4, 3)


def test_two_by_two_hand_moments():
    maps = bm.sliding_moments(np.array([[0.0, 1.0], [2.0, 3.0]]), window=(2, 2))
    assert maps.shape == (1, 1)
    assert (maps.m1[0, 0], maps.m2[0, 0], maps.m3[0, 0]) == (1.5, 3.5, 9.0)


def test_window_equal_to_image_gives_whole_image_moments():
    img = np.random.default_rng(0).random((7, 5))
    maps = bm.sliding_moments(img, window=(7, 5))
    assert maps.m1[0, 0] == pytest.approx(img.mean(), rel=1e-15)
    assert maps.m2[0, 0] == pytest.approx((img**2).mean(), rel=1e-15)


def test_moment_grid_dims_and_errors():
    maps = bm.sliding_moments(np.zeros((20, 13)), window=(4, 3), stride=(3, 2))
    assert maps.shape == ((20 - 4) // 3 + 1, (13 - 3) // 2 + 1)
    with pytest.raises(WindowTooLarge):
        bm.sliding_moments(np.zeros((4, 4)), window=(5, 2))
    with pytest.raises(DimensionMismatch):
        bm.sliding_moments(np.zeros((4, 4, 2)), window=(2, 2))
    with pytest.raises(InvalidMetadata):
        bm.sliding_moments(np.zeros((4, 4)), window=(2, 2), stride=(0, 1))


def test_variance_nonnegative_on_random_fields():
    rng = np.random.default_rng(1)
    for _ in range(20):
        img = rng.rayleigh(1.0, size=(32, 32))
        maps = bm.sliding_moments(img, window=(5, 5), stride=(3, 3))
        assert np.all(maps.m2 - maps.m1**2 >= -1e-12 * np.maximum(maps.m2, 1.0))
        assert np.all(maps.m2 >= 0) and np.all(maps.m3 >= 0)


def test_criterion_7_statistical_moments():
    field = np.random.default_rng(123).rayleigh(scale=1.0, size=(1000, 1000))
    maps = bm.sliding_moments(field, window=field.shape)
    assert abs(maps.m2[0, 0] - 2.0) < 0.02
    assert maps.m2[0, 0] == pytest.approx((field**2).mean(), rel=1e-13)
    const = bm.sliding_moments(np.full((64, 64), 2.0), window=(8, 8), stride=(4, 4))
    np.testing.assert_array_equal(const.m1, 2.0)
    np.testing.assert_array_equal(const.m2, 4.0)
    np.testing.assert_array_equal(const.m3, 8.0)


def test_dense_forward_hand_cases():
    trunc = bm.DenseModel((bm.DenseLayer(np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]]),
                                         np.zeros(2), "identity"),))
    np.testing.assert_array_equal(bm.dense_forward([1.0, 2.0, 3.0], trunc), [1.0, 2.0])
    np.testing.assert_array_equal(bm.dense_forward([1.0, 2.0, 3.0], one_layer_model()),
                                  [6.0, 4.0])
    relu = bm.DenseModel((bm.DenseLayer(np.array([[-1.0, 0.0, 0.0], [0.0, 0.0, 1.0]]),
                                        np.zeros(2), "relu"),))
    np.testing.assert_array_equal(bm.dense_forward([1.0, 0.0, 5.0], relu), [0.0, 5.0])


def test_relu_positive_homogeneity_and_softplus_sign():
    rng = np.random.default_rng(2)
    model = bm.DenseModel((bm.DenseLayer(rng.normal(size=(5, 3)), np.zeros(5), "relu"),
                           bm.DenseLayer(rng.normal(size=(2, 5)), np.zeros(2), "relu")))
    x = rng.normal(size=3)
    np.testing.assert_allclose(bm.dense_forward(3.0 * x, model),
                               3.0 * bm.dense_forward(x, model), rtol=1e-12)
    rng = np.random.default_rng(3)
    sp = bm.DenseModel((bm.DenseLayer(rng.normal(size=(2, 3)), rng.normal(size=2),
                                      "softplus"),))
    out = bm.dense_forward(rng.normal(size=(10, 3)), sp)
    assert out.shape == (10, 2) and np.all(out >= 0)
    z = np.array([[0.0, 0.0, 0.0]])  # softplus(0) = log 2 (logaddexp's x == y branch)
    zero = bm.DenseModel((bm.DenseLayer(np.zeros((2, 3)), np.zeros(2), "softplus"),))
    np.testing.assert_array_equal(bm.dense_forward(z, zero), np.log(2.0))


def test_dense_forward_width_checked():
    with pytest.raises(DimensionMismatch):
        bm.dense_forward([1.0, 2.0], one_layer_model())


def test_estimate_map_hand_and_constant_cases():
    hk = bm.estimate_hk_map(np.array([[0.0, 1.0], [2.0, 3.0]]), window=(2, 2), stride=(1, 1),
                            model=one_layer_model())
    assert (hk.u[0, 0], hk.k[0, 0]) == (14.0, 10.0)
    rng = np.random.default_rng(4)
    model = bm.DenseModel((bm.DenseLayer(rng.normal(size=(4, 3)), rng.normal(size=4), "relu"),
                           bm.DenseLayer(rng.normal(size=(2, 4)), rng.normal(size=2),
                                         "identity")))
    hk = bm.estimate_hk_map(np.full((12, 12), 1.7), window=(4, 4), stride=(2, 2), model=model)
    np.testing.assert_allclose(hk.u, hk.u[0, 0])
    np.testing.assert_allclose(hk.k, hk.k[0, 0])
    zero = bm.DenseModel((bm.DenseLayer(np.zeros((2, 3)), np.array([0.5, -1.5]), "relu"),))
    hk = bm.estimate_hk_map(np.ones((6, 6)), window=(3, 3), stride=(1, 1), model=zero)
    np.testing.assert_array_equal(hk.u, 0.5)
    np.testing.assert_array_equal(hk.k, 0.0)


def test_estimate_equals_mapped_dense_forward():
    rng = np.random.default_rng(5)
    model = bm.DenseModel((
        bm.DenseLayer(rng.normal(size=(4, 3)), rng.normal(size=4), "softplus"),
        bm.DenseLayer(rng.normal(size=(2, 4)), rng.normal(size=2), "identity")))
    img = rng.rayleigh(1.0, size=(16, 14))
    window, stride = (5, 4), (2, 3)
    maps = bm.sliding_moments(img, window, stride)
    hk = bm.estimate_hk_map(img, window, stride, model)
    uk = bm.dense_forward(maps.stacked(), model)
    np.testing.assert_allclose(hk.u, uk[..., 0], rtol=1e-12)
    np.testing.assert_allclose(hk.k, uk[..., 1], rtol=1e-12)


def test_device_envelope_input_and_pipeline_nodes(tmp_path):
    """Envelope images stay on the GPU up to the QUS nodes: the moments node
    and a model-file hk_estimator node run after `envelope` in a chain."""
    import torch

    env = torch.from_numpy(np.random.default_rng(8).rayleigh(1.0, size=(64, 32))).cuda()
    maps = bm.sliding_moments(env, (8, 4), (4, 2))
    ref = bm.sliding_moments(env.cpu().numpy(), (8, 4), (4, 2))
    np.testing.assert_array_equal(maps.m1, ref.m1)

    path = tmp_path / "m.hkdm"
    bm.save_model(one_layer_model(), path)
    spec = bm.bmode_chain()
    spec["nodes"] += [
        {"name": "moments", "kind": "sliding_moments",
         "params": {"window": [64, 4], "stride": [32, 2]}},
        {"name": "hk", "kind": "hk_estimator",
         "params": {"window": [64, 4], "stride": [32, 2], "model_path": str(path)}}]
    spec["edges"] += [{"from": "envelope", "to": "moments"}, {"from": "envelope", "to": "hk"}]
    spec["outputs"] = ["dynamic_adjustment", "moments", "hk"]
    graph = bm.build_graph(spec)
    ctx, grid, n_s = bm.environment.config_geometry("cfg1", n_z=64, n_x=16, n_tx=16, n_el=16)
    frame = bm.RfFrame(np.random.default_rng(1).normal(size=(ctx.n_tx, 16, 512))
                       .astype(np.float32))
    outputs, _ = bm.execute(graph, (frame, ctx))
    maps = outputs["moments"]
    assert maps.shape == ((512 - 64) // 32 + 1, (16 - 4) // 2 + 1)
    assert np.all(maps.m2 >= 0)
    hk = outputs["hk"]
    np.testing.assert_allclose(hk.u, maps.m1 + maps.m2 + maps.m3, rtol=1e-12)
    np.testing.assert_allclose(hk.k, maps.m3 + 1.0, rtol=1e-12)
