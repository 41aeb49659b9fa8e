"""Host half of the QUS hooks (no GPU): model validation and the model file
format, ported from the reference's test_qus.py:97-206 and qus.py:1-19."""

import numpy as np
import pytest

import paper_1811_01566_b200 as bm
from paper_1811_01566_b200.errors import DimensionMismatch, FormatError, InvalidMetadata


def one_layer_model():
    return bm.DenseModel((bm.DenseLayer(np.array([[1.0, 1.0, 1.0], [0.0, 0.0, 1.0]]),
                                        np.array([0.0, 1.0]), "identity"),))


def test_model_dimension_chain_checked():
    with pytest.raises(DimensionMismatch):
        bm.DenseModel((bm.DenseLayer(np.zeros((4, 3)), np.zeros(4), "relu"),
                       bm.DenseLayer(np.zeros((2, 5)), np.zeros(2), "identity")))
    with pytest.raises(DimensionMismatch):
        bm.DenseModel((bm.DenseLayer(np.zeros((2, 4)), np.zeros(2), "identity"),))
    with pytest.raises(DimensionMismatch):
        bm.DenseModel((bm.DenseLayer(np.zeros((3, 3)), np.zeros(3), "identity"),))
    with pytest.raises(InvalidMetadata):
        bm.DenseModel(())
    with pytest.raises(InvalidMetadata):
        bm.DenseLayer(np.zeros((2, 3)), np.zeros(2), "tanh")
    with pytest.raises(InvalidMetadata):
        bm.DenseLayer(np.full((2, 3), np.nan), np.zeros(2), "relu")


def test_moment_maps_validation():
    z = np.zeros((2, 2))
    with pytest.raises(InvalidMetadata):
        bm.MomentMaps(z, -np.ones((2, 2)), z, (1, 1), (1, 1))
    with pytest.raises(InvalidMetadata):  # variance below the slack
        bm.MomentMaps(np.full((2, 2), 2.0), np.full((2, 2), 3.0), z, (1, 1), (1, 1))
    with pytest.raises(DimensionMismatch):
        bm.MomentMaps(z, np.zeros((3, 2)), z, (1, 1), (1, 1))


def test_model_file_round_trip(tmp_path):
    rng = np.random.default_rng(6)
    model = bm.DenseModel((
        bm.DenseLayer(rng.normal(size=(8, 3)), rng.normal(size=8), "relu"),
        bm.DenseLayer(rng.normal(size=(4, 8)), rng.normal(size=4), "relu"),
        bm.DenseLayer(rng.normal(size=(2, 4)), rng.normal(size=2), "softplus"),
    ))
    path = tmp_path / "model.hkdm"
    bm.save_model(model, path)
    blob = path.read_bytes()
    assert blob.startswith(b"HKDM 1\nlayers 3\n3 8 relu\n8 4 relu\n4 2 softplus\nend\n")
    back = bm.load_model(path)
    assert len(back.layers) == 3
    for a, b in zip(model.layers, back.layers):
        np.testing.assert_array_equal(a.weights, b.weights)
        np.testing.assert_array_equal(a.bias, b.bias)
        assert a.activation == b.activation


def test_model_file_written_by_reference_layout_loads(tmp_path):
    """Header + little-endian f64 payload, byte for byte as qus.py:1-19 documents."""
    w = np.array([[1.0, 1.0, 1.0], [0.0, 0.0, 1.0]])
    b = np.array([0.0, 1.0])
    path = tmp_path / "hand.hkdm"
    path.write_bytes(b"HKDM 1\nlayers 1\n3 2 identity\nend\n" + w.astype("<f8").tobytes()
                     + b.astype("<f8").tobytes())
    m = bm.load_model(path)
    np.testing.assert_array_equal(m.layers[0].weights, w)
    np.testing.assert_array_equal(m.layers[0].bias, b)


@pytest.mark.parametrize("blob,where", [
    (b"XXXX 1\nlayers 1\n3 2 identity\nend\n" + b"\x00" * 64, "bad magic"),
    (b"HKDM 2\nlayers 1\n3 2 identity\nend\n" + b"\x00" * 64, "unsupported version"),
    (b"HKDM 1\nlayers 1\n3 2 tanh\nend\n" + b"\x00" * 64, "unknown activation"),
    (b"HKDM 1\nlayers x\n", "not an integer"),
    (b"HKDM 1\nlayers 0\n", "must be >= 1"),
    (b"HKDM 1\nlayers 1\n3 2\nend\n", "expected '<in> <out> <activation>'"),
    (b"HKDM 1\nlayers 1\n3 2 identity\nfin\n", "expected 'end'"),
    (b"HKDM 1\nlayers 1\n3 2 identity", "truncated header"),
    (b"HKDM 1\nlayers 1\n3 2 identity\nend\n" + b"\x00" * 64 + b"\x00", "trailing bytes"),
    (b"HKDM 1\nlayers 1\n3 3 identity\nend\n" + b"\x00" * 96, "inconsistent model"),
])
def test_model_file_defects(tmp_path, blob, where):
    path = tmp_path / "bad.hkdm"
    path.write_bytes(blob)
    with pytest.raises(FormatError) as err:
        bm.load_model(path)
    assert where in str(err.value)


def test_model_file_truncated_payload(tmp_path):
    path = tmp_path / "m.hkdm"
    bm.save_model(one_layer_model(), path)
    (tmp_path / "cut.hkdm").write_bytes(path.read_bytes()[:-8])
    with pytest.raises(FormatError) as err:
        bm.load_model(tmp_path / "cut.hkdm")
    assert "truncated" in str(err.value)
