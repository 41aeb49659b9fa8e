"""GPU: the full Fig-2 chain through the operator registry (bmode_chain ->
build_graph -> execute) against the reference's chain outputs, and the
reference's pipeline-level behaviours (test_pipeline.py / test_acceptance.py)."""

import os

import numpy as np
import pytest

import cases
import paper_1811_01566_b200 as bm
from paper_1811_01566_b200.errors import OperatorFailed

pytestmark = pytest.mark.gpu

# f32 chain tolerances vs the reference (DAS is bitwise; FFT is not):
ENV_REL = 2e-6   # max|d env| / max env
DISP_ABS = 2e-5  # display units ([0, 1]); ~6e-4 dB of a 30 dB range


def run_chain(ctx, data, grid, apod, interp):
    spec = bm.bmode_chain(window=apod.window, f_number=apod.f_number, interpolation=interp,
                          grid={"x_positions": grid.x_positions.tolist(),
                                "z_positions": grid.z_positions.tolist()})
    spec["outputs"] = ["beamform", "envelope", "dynamic_adjustment"]
    graph = bm.build_graph(spec)
    outs, timing = bm.execute(graph, (bm.RfFrame(data), ctx))
    return outs, timing


def test_chain_vs_reference(golden_dir):
    g = np.load(os.path.join(golden_dir, "chain.npz"))
    for name, ctx, data, grid, apod, interp in cases.chain_cases(bm.types):
        outs, timing = run_chain(ctx, data, grid, apod, interp)
        rf = outs["beamform"].numpy()
        env = outs["envelope"].numpy()
        disp = outs["dynamic_adjustment"].numpy()
        assert rf.tobytes() == g[f"{name}_rf"].tobytes(), name
        ref_env = g[f"{name}_env"]
        assert np.abs(env - ref_env).max() <= ENV_REL * ref_env.max(), name
        assert disp.dtype == np.float32
        assert np.abs(disp - g[f"{name}_disp"]).max() <= DISP_ABS, name
        assert disp.max() == 1.0 and disp.min() >= 0.0
        assert [s for s, _ in timing.stages] == ["beamform", "analytic_signal", "envelope",
                                                 "dynamic_adjustment"]
        assert all(ms >= 0 for _, ms in timing.stages)


def test_deferred_analytic_materialises(golden_dir):
    g = np.load(os.path.join(golden_dir, "chain.npz"))
    name, ctx, data, grid, apod, interp = cases.chain_cases(bm.types)[0]
    spec = bm.bmode_chain(grid={"x_positions": grid.x_positions.tolist(),
                                "z_positions": grid.z_positions.tolist()})
    spec["outputs"] = ["analytic_signal", "dynamic_adjustment"]
    outs, _ = bm.execute(bm.build_graph(spec), (bm.RfFrame(data), ctx))
    z = outs["analytic_signal"].data.cpu().numpy()
    ref = g[f"{name}_z"]
    assert np.abs(z - ref).max() <= 2e-6 * np.abs(ref).max()


def test_all_zero_frame_fails_in_dynamic_adjustment():
    ctx = bm.AcquisitionContext(1540.0, 40e6, 8, 2e-4, bm.StaScheme(tuple(range(8))))
    graph = bm.build_graph(bm.bmode_chain())
    with pytest.raises(OperatorFailed) as err:
        bm.execute(graph, (bm.RfFrame(np.zeros((8, 8, 256))), ctx))
    assert err.value.node == "dynamic_adjustment"


def test_localization_sta_and_pw():
    """Criterion 3 (test_acceptance.py:90-121): the envelope argmax of a
    simulated point scatterer lands within +/-1 cell for STA and PW."""
    scat = (0.45e-3, 14.2e-3)
    ph = bm.Phantom(((scat[0], scat[1], 1.0),), center_frequency=5e6, n_cycles=2)
    for scheme in ("sta", "pw"):
        tx = (bm.StaScheme(tuple(range(32))) if scheme == "sta"
              else bm.PwScheme(tuple(bm.default_pw_angles())))
        ctx = bm.AcquisitionContext(1540.0, 40e6, 32, 2e-4, tx)
        frame = bm.simulate_rf(ph, ctx, 1024)
        grid = bm.default_grid(ctx, 1024, scheme)
        img = bm.das_beamform(frame, ctx, grid)
        env = bm.envelope(bm.analytic_signal(img.data, axis=0))
        iz, ix = np.unravel_index(env.argmax(), env.shape)
        assert abs(iz - np.abs(grid.z_positions - scat[1]).argmin()) <= 1
        assert abs(ix - np.abs(grid.x_positions - scat[0]).argmin()) <= 1


def test_seeded_benchmark_outputs_identical():
    ph = bm.Phantom(((0.2e-3, 6e-3, 1.0),), center_frequency=5e6, n_cycles=2)
    ctx = bm.AcquisitionContext(1540.0, 40e6, 24, 2e-4, bm.StaScheme(tuple(range(24))))
    graph = bm.build_graph(bm.bmode_chain())

    def run():
        env = bm.open_simulator(ph, ctx, 512, seed=11, noise_std=0.1)
        return bm.benchmark(graph, env, n_frames=2, warmup=1, keep_outputs=True)

    r1, r2 = run(), run()
    for o1, o2 in zip(r1.outputs, r2.outputs):
        assert (o1["dynamic_adjustment"].numpy().tobytes()
                == o2["dynamic_adjustment"].numpy().tobytes())
    assert r1.timing.total_ms > 0


def test_staged_host_to_device_copies_are_exact_and_do_not_alias():
    """Large numpy inputs reach the device through two alternating pinned
    staging buffers (_device._staged_h2d): every copy is exact, and a later
    copy never overwrites the data of an earlier one still in flight."""
    import torch

    from paper_1811_01566_b200._device import to_device

    rng = np.random.default_rng(3)
    dev = torch.device("cuda", 0)
    hosts = [rng.normal(size=(11, 128, 512)).astype(np.float32) for _ in range(5)]
    outs = [to_device(h, dev) for h in hosts]          # 2.9 MB each: staged
    small = to_device(hosts[0][:1, :1], dev)            # below the threshold: plain copy
    torch.cuda.synchronize()
    for h, o in zip(hosts, outs):
        assert torch.equal(o.cpu(), torch.from_numpy(h))
    assert torch.equal(small.cpu(), torch.from_numpy(hosts[0][:1, :1].copy()))
    f64 = to_device(hosts[1].astype(np.float64), dev)
    assert f64.dtype == torch.float64 and torch.equal(f64.cpu(), torch.from_numpy(hosts[1].astype(np.float64)))


def test_host_upload_pieces_counter_and_odd_sizes():
    """bm_host_upload: byte-exact for odd sizes and unaligned source /
    destination offsets, empty pieces allowed, the counter ends at the last
    piece's value; bad arguments rejected before any work."""
    import ctypes

    import torch

    from paper_1811_01566_b200 import _native as N

    rng = np.random.default_rng(9)
    lib = N.load()
    st = torch.cuda.current_stream()
    counter = torch.zeros(1, dtype=torch.int32, device="cuda")
    for nbytes, cuts in ((1, [1]), (1000, [0, 999, 1000]), (3 << 20, [1 << 20, 1 << 20, 3 << 20]),
                         ((5 << 20) + 13, [7, (2 << 20) + 1, (5 << 20) + 13])):
        src = rng.integers(0, 256, size=nbytes + 3, dtype=np.uint8)
        stage = torch.empty(nbytes + 64, dtype=torch.uint8, pin_memory=True)
        dst = torch.zeros(nbytes + 5, dtype=torch.uint8, device="cuda")
        ends = (ctypes.c_int64 * len(cuts))(*cuts)
        vals = (ctypes.c_uint32 * len(cuts))(*[100 + i for i in range(len(cuts))])
        # odd offsets: source +3, staging +1, destination +5
        N.call("bm_host_upload", dst.data_ptr() + 5, src.ctypes.data + 3, stage.data_ptr() + 1,
               ends, len(cuts), counter.data_ptr(), vals, st.cuda_stream)
        torch.cuda.synchronize()
        assert np.array_equal(dst[5:].cpu().numpy(), src[3:]), nbytes
        assert int(counter.item()) == 100 + len(cuts) - 1
    bad = (ctypes.c_int64 * 2)(8, 4)  # decreasing ends
    assert lib.bm_host_upload(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src.ctypes.data),
                              ctypes.c_void_p(stage.data_ptr()), bad, 2, None, None,
                              ctypes.c_void_p(st.cuda_stream)) == 1


def test_device_frame_finiteness_scan_on_the_gpu():
    """RfFrame of a CUDA tensor runs the reference's finiteness check
    (types.py:41-42) with bm_check_finite: NaN and inf rejected."""
    import torch

    from paper_1811_01566_b200.errors import InvalidMetadata

    x = torch.randn(3, 4, 257, device="cuda")
    bm.RfFrame(x)
    for bad in (float("nan"), float("inf"), -float("inf")):
        y = x.clone()
        y[2, 3, 256] = bad
        with pytest.raises(InvalidMetadata):
            bm.RfFrame(y)
        with pytest.raises(InvalidMetadata):
            bm.RfFrame(y.double())


def test_stage_times_bracket_each_ops_gpu_work():
    """execute's CUDA-event stage times hold each node's own GPU work: the
    beamform stage of the sta-paper preset is at least most of the same op
    timed alone (an event on the wrong stream would leave the DAS outside
    it and charge it to a later stage)."""
    import statistics

    import torch

    from paper_1811_01566_b200 import cli
    from paper_1811_01566_b200.pipeline import _to_device_obs

    env = cli.preset_environment("sta-paper")
    g = bm.build_graph(cli.preset_pipeline("sta-paper"))
    obs = _to_device_obs(env.next_observation())
    for _ in range(3):
        bm.execute(g, obs)
    stage = statistics.median(bm.execute(g, obs)[1].stage_ms("beamform") for _ in range(5))
    node = g.nodes["beamform"].fn
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    alone = []
    for _ in range(5):
        torch.cuda.synchronize()
        a.record()
        node(obs)
        b.record()
        torch.cuda.synchronize()
        alone.append(a.elapsed_time(b))
    assert stage >= 0.6 * statistics.median(alone), (stage, alone)
