"""CPU: pin the oracle (oracle/) to fixtures generated from the reference
itself (tests/golden/make_golden.py).  DAS parity is bitwise."""

import hashlib
import json
import os

import numpy as np
import pytest

import cases
from oracle import oracle as O
from paper_1811_01566_b200 import environment as ME
from paper_1811_01566_b200 import types as T


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def small(golden_dir):
    z = np.load(os.path.join(golden_dir, "das_small.npz"))
    return z, dict(zip(z["hash_keys"].tolist(), z["hash_vals"].tolist()))


def test_criterion4_oracle_bitwise_vs_reference(small):
    _, hashes = small
    n = 0
    for i, (ctx, data, grid, apod) in enumerate(cases.criterion4_cases(T)):
        for dt in ("f64", "f32"):
            x = data if dt == "f64" else data.astype(np.float32)
            for interp in ("nearest", "linear"):
                img = O.das_beamform(x, ctx, grid, apod.window, apod.f_number, interp,
                                     n_threads=2)
                assert sha(img) == hashes[f"{i}_{dt}_{interp}"], (i, dt, interp)
                n += 1
    assert n == 400


def test_direct_oracle_matches_reference_oracle(small):
    z, _ = small
    for i, (ctx, data, grid, apod) in enumerate(cases.criterion4_cases(T, n_cases=12)):
        d = O.das_beamform_direct(data, ctx, grid, apod.window, apod.f_number, "linear")
        assert d.tobytes() == z[f"{i}_f64_linear_oracle"].tobytes(), i


def test_chain_oracle_vs_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "chain.npz"))
    for name, ctx, data, grid, apod, interp in cases.chain_cases(T):
        rf, env, disp = O.bmode_chain(data, ctx, grid, apod.window, apod.f_number, interp)
        assert rf.tobytes() == g[f"{name}_rf"].tobytes(), name
        np.testing.assert_array_equal(env, g[f"{name}_env"])
        np.testing.assert_array_equal(disp, g[f"{name}_disp"])
        rf64, _, disp64 = O.bmode_chain(data.astype(np.float64), ctx, grid, apod.window,
                                        apod.f_number, interp)
        assert rf64.tobytes() == g[f"{name}_rf64"].tobytes(), name
        np.testing.assert_array_equal(disp64, g[f"{name}_disp64"])


def test_sigproc_oracle_vs_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "sigproc.npz"))
    for n in (2, 3, 8, 9, 33, 64, 100, 256, 1000, 1024):
        np.testing.assert_array_equal(O.analytic_signal(g[f"x32_{n}"], axis=0), g[f"z32_{n}"])
        np.testing.assert_array_equal(O.analytic_signal(g[f"x64_{n}"], axis=0), g[f"z64_{n}"])
    np.testing.assert_array_equal(O.dynamic_adjustment(g["dyn_in32"], 30.0), g["dyn_out32_30"])
    np.testing.assert_array_equal(O.dynamic_adjustment(g["dyn_in32"], 45.0), g["dyn_out32_45"])
    np.testing.assert_array_equal(O.dynamic_adjustment(g["dyn_in64"], 30.0), g["dyn_out64_30"])


@pytest.mark.parametrize("key", ["cfg1_f32_linear_seed0", "cfg1_f32_nearest_seed0",
                                 "cfg1_f64_linear_seed0", "cfg2_f32_linear_seed1"])
def test_full_size_oracle_hash(golden_dir, key):
    ref = json.load(open(os.path.join(golden_dir, "configs.json")))
    name, dt, interp, seed = key.split("_")
    ctx, grid, n_s = ME.config_geometry(name)
    data = cases.config_rf((ctx.n_tx, ctx.n_elements, n_s), int(seed[4:]))
    if dt == "f64":
        data = data.astype(np.float64)
    img = O.das_beamform(data, ctx, grid, interp=interp)
    assert sha(img) == ref[key]


def test_simulator_restatement_matches_reference(golden_dir):
    ref = json.load(open(os.path.join(golden_dir, "configs.json")))
    ctx, grid, n_s = ME.config_geometry("cfg2")
    env = ME.open_simulator(ME.wire_phantom(), ctx, n_s, dtype=np.float32, seed=0,
                            noise_std=0.01)
    frame, _ = env.next_observation()
    assert sha(frame.data) == ref["sim_cfg2_wire_f32_seed0_noise0.01"]


def test_oracle_thread_count_bits():
    ctx, grid, n_s = ME.config_geometry("cfg1", n_z=64, n_x=64, n_tx=64)
    data = cases.config_rf((ctx.n_tx, ctx.n_elements, n_s), 3)
    a = O.das_beamform(data, ctx, grid, n_threads=1)
    b = O.das_beamform(data, ctx, grid, n_threads=3)
    assert a.tobytes() == b.tobytes()


def test_fir_oracle_matches_reference_goldens(golden_dir):
    """oracle.fir_filter (np.convolve in f64, lfilter's one-term-denominator
    branch) reproduces the reference's fir_filter bits."""
    g = np.load(os.path.join(golden_dir, "fir.npz"))
    for nt in (1, 2, 7, 33, 64):
        h = g[f"h_{nt}"]
        for xk, yk, ax in (("x32", "y32", -1), ("x64", "y64", -1), ("xa", "ya", 0)):
            y = O.fir_filter(g[f"{xk}_{nt}"], h, axis=ax)
            ref = g[f"{yk}_{nt}"]
            assert y.dtype == ref.dtype == np.float64
            assert np.array_equal(y, ref), (nt, xk)


def test_qus_oracle_matches_reference_goldens(golden_dir):
    """oracle.sliding_moments / dense_forward reproduce the reference's
    qus outputs bit for bit (same numpy operations)."""
    g = np.load(os.path.join(golden_dir, "qus.npz"))
    layers = [(g[f"W_{j}"], g[f"b_{j}"], str(a)) for j, a in enumerate(g["acts"])]
    for i in range(4):
        m1, m2, m3 = O.sliding_moments(g[f"img_{i}"], tuple(g[f"win_{i}"]), tuple(g[f"stride_{i}"]))
        assert np.array_equal(m1, g[f"m1_{i}"]) and np.array_equal(m2, g[f"m2_{i}"])
        assert np.array_equal(m3, g[f"m3_{i}"])
        out = O.dense_forward(np.stack([m1, m2, m3], axis=-1), layers)
        assert np.array_equal(out[..., 0], g[f"u_{i}"]) and np.array_equal(out[..., 1], g[f"k_{i}"])


def test_host_simulator_matches_reference_sim_goldens(golden_dir):
    """The host restatement of simulate_rf (the bench's input generator and
    the GPU simulator's checker) reproduces the reference bit for bit."""
    g = np.load(os.path.join(golden_dir, "sim.npz"))
    ph = ME.Phantom(((0.4e-3, 4.9e-3, 1.0), (-1.1e-3, 7.3e-3, 0.6), (2.0e-3, 3.1e-3, -0.8)),
                    center_frequency=5e6, n_cycles=2)
    ctx = T.AcquisitionContext(1540.0, 40e6, 16, 2e-4, T.StaScheme((0, 5, 11, 15)),
                               rx_channel_map=np.array([[i, (i + 3) % 16, 15 - i]
                                                        for i in (0, 5, 11, 15)]),
                               time_zero_offset=np.array([0.0, 1e-7, -2e-7, 3.3e-7]))
    assert np.array_equal(ME.simulate_rf(ph, ctx, 600, np.float64).data, g["sta_f64"])
    ctx = T.AcquisitionContext(1480.0, 31.25e6, 24, 3e-4, T.PwScheme((-0.2, 0.05, 0.17)))
    assert np.array_equal(ME.simulate_rf(ph, ctx, 500, np.float64).data, g["pw_f64"])
    ctx, grid, n_s = ME.config_geometry("cfg2")
    clean = ME.simulate_rf(ME.wire_phantom(), ctx, n_s, np.float32).data
    assert hashlib.sha256(clean.tobytes()).hexdigest() == str(g["cfg2_wire_f32_sha256"])
