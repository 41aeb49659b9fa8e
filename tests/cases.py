"""Seeded test-case generators shared by the golden-fixture script and the
tests.  ``T`` is a types module: echopipe.types when make_golden.py runs the
reference, paper_1811_01566_b200.types in the tests.  The draw order is
identical in both, so the same seed yields the same instances."""

from __future__ import annotations

import numpy as np


def criterion4_cases(T, seed=2024, n_cases=100):
    """Replays the randomized instance generator of the reference's criterion-4
    acceptance test (test_acceptance.py:124-177): n_el, n_rx <= 8, n_tx <= 8,
    16..256 samples, random STA/PW, rx map, t0 and apodisation, 16x16 grid."""
    rng = np.random.default_rng(seed)
    for _ in range(n_cases):
        n_el = int(rng.integers(1, 9))
        n_rx = int(rng.integers(1, n_el + 1))
        n_tx = int(rng.integers(1, 9))
        n_samples = int(rng.integers(16, 257))
        pitch = float(rng.uniform(1e-4, 4e-4))
        fs = float(rng.uniform(10e6, 50e6))
        if rng.random() < 0.5:
            scheme = T.StaScheme(tuple(rng.integers(0, n_el, size=n_tx)))
        else:
            scheme = T.PwScheme(tuple(rng.uniform(-0.3, 0.3, size=n_tx)))
        rx_map = None
        if n_rx != n_el or rng.random() < 0.3:
            rx_map = rng.integers(0, n_el, size=(n_tx, n_rx))
        ctx = T.AcquisitionContext(
            speed_of_sound=float(rng.uniform(1400, 1600)), sampling_frequency=fs,
            n_elements=n_el, pitch=pitch, tx_scheme=scheme, rx_channel_map=rx_map,
            time_zero_offset=rng.normal(scale=2e-7, size=n_tx))
        data = rng.normal(size=(n_tx, n_rx, n_samples))
        span = n_el * pitch
        grid = T.ImageGrid(np.linspace(-span, span, 16),
                           np.linspace(1e-4, n_samples / fs * ctx.speed_of_sound / 2, 16))
        apod = T.ApodizationSpec(window=("rectangular", "hann")[int(rng.random() < 0.5)],
                                 f_number=float(rng.choice([0.0, 0.8, 2.0])))
        yield ctx, data, grid, apod


def chain_cases(T):
    """Mid-size Fig-2 chain instances (f32) covering STA/PW, rx maps, t0,
    Hann + f-number and both interpolations.  RF is seeded white noise plus
    a few impulses, so no simulator is needed to rebuild it."""
    out = []
    c, fs = 1540.0, 40e6

    def rf(seed, shape):
        r = np.random.default_rng(seed)
        x = 0.01 * r.normal(size=shape)
        for _ in range(6):
            e, j, k = (int(r.integers(0, s)) for s in shape)
            x[e, j, max(0, k - 3):k + 3] += np.hanning(8)[: len(x[e, j, max(0, k - 3):k + 3])]
        return x.astype(np.float32)

    # STA, identity map, rectangular F=0 (the benchmark form), linear
    ctx = T.AcquisitionContext(c, fs, 16, 2e-4, T.StaScheme(tuple(range(16))))
    ex = ctx.element_positions()
    grid = T.ImageGrid(np.linspace(ex[0], ex[-1], 48), np.linspace(0, 512 * c / (2 * fs), 64))
    out.append(("sta_rect_linear", ctx, rf(1, (16, 16, 512)), grid,
                T.ApodizationSpec(), "linear"))
    # STA nearest, Hann F=1.5, t0 per acquisition
    ctx = T.AcquisitionContext(c, fs, 16, 2e-4, T.StaScheme(tuple(range(16))),
                               time_zero_offset=np.linspace(-2e-7, 3e-7, 16))
    out.append(("sta_hann_nearest", ctx, rf(2, (16, 16, 512)), grid,
                T.ApodizationSpec("hann", 1.5), "nearest"))
    # STA with a centred 8-of-24 rx map (paper STA convention), linear, rect F=1
    tx = tuple(range(0, 24, 2))
    ctx = T.AcquisitionContext(c, fs, 24, 2e-4, T.StaScheme(tx),
                               rx_channel_map=T.centered_rx_map(24, 8, tx))
    ex = ctx.element_positions()
    grid2 = T.ImageGrid(np.linspace(ex[0], ex[-1], 40), np.linspace(1e-3, 600 * c / (2 * fs), 72))
    out.append(("sta_map_rectF1_linear", ctx, rf(3, (12, 8, 600)), grid2,
                T.ApodizationSpec("rectangular", 1.0), "linear"))
    # PW, 5 angles, 32 elements, linear rect F=0 and Hann F=2 nearest
    ang = tuple(np.deg2rad([-8.0, -4.0, 0.0, 4.0, 8.0]))
    ctx = T.AcquisitionContext(c, fs, 32, 2e-4, T.PwScheme(ang))
    ex = ctx.element_positions()
    grid3 = T.ImageGrid(np.linspace(ex[0], ex[-1], 64), np.linspace(0, 512 * c / (2 * fs), 80))
    out.append(("pw_rect_linear", ctx, rf(4, (5, 32, 512)), grid3, T.ApodizationSpec(), "linear"))
    out.append(("pw_hann_nearest", ctx, rf(5, (5, 32, 512)), grid3,
                T.ApodizationSpec("hann", 2.0), "nearest"))
    # PW with t0 offsets and odd image height (general-N analytic signal)
    ctx = T.AcquisitionContext(c, 20e6, 20, 3e-4, T.PwScheme(tuple(np.deg2rad([-5.0, 0.0, 7.0]))),
                               time_zero_offset=np.array([1e-7, 0.0, -1e-7]))
    ex = ctx.element_positions()
    grid4 = T.ImageGrid(np.linspace(ex[0], ex[-1], 33), np.linspace(5e-4, 300 * 1540 / 40e6, 75))
    out.append(("pw_t0_oddN_linear", ctx, rf(6, (3, 20, 300)), grid4,
                T.ApodizationSpec("hann", 0.8), "linear"))
    return out


def config_rf(shape, seed, kind="noise"):
    """Full-size synthetic RF that any box can regenerate: seeded N(0,1) f32."""
    return np.random.default_rng(seed).normal(size=shape).astype(np.float32)


# (n, f32 lanes, f64 lanes) of the long-axis analytic-signal goldens: 37 lanes
# leave a partial 8-lane CTA
LONG_AXES = ((2048, 37, 5), (4096, 9, 3))


def long_lanes(n, lanes, dtype):
    """Seeded [n, lanes] input of the long-axis analytic-signal goldens."""
    return np.random.default_rng(1000 + 7 * n + lanes).normal(size=(n, lanes)).astype(dtype)
