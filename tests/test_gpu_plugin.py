"""The drop-in proven where a reference user meets it: echopipe's OWN graph
builder, executor and benchmark (baseline/_ref, the vendored reference
install) running the B200 kinds registered through its own
``register_operator`` (pipeline.py:63-77).

Checked against the reference's own chain outputs (tests/golden/chain.npz):
beamformed RF bitwise, display <= 2e-5.  Under echopipe's per-node
perf_counter (pipeline.py:369-381) each stage's time must be its own: the
synchronous op wrappers make every node return after its GPU work."""

import os
import sys

import numpy as np
import pytest

import cases
import paper_1811_01566_b200 as bm

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


@pytest.fixture(scope="module")
def ep():
    if not os.path.isdir(os.path.join(REF, "echopipe")):
        pytest.skip("baseline/_ref/echopipe (the vendored reference install) is absent")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_echopipe")
    sys.path.insert(0, REF)
    import echopipe
    import echopipe.pipeline as EPL

    saved = dict(EPL.OPERATOR_REGISTRY)
    bm.register_gpu_operators(register=EPL.register_operator)
    yield echopipe
    EPL.OPERATOR_REGISTRY.clear()
    EPL.OPERATOR_REGISTRY.update(saved)


def _host(x):
    return x.numpy() if hasattr(x, "numpy") and not isinstance(x, np.ndarray) else np.asarray(x)


def test_echopipe_execute_runs_the_b200_kinds(ep, golden_dir):
    import echopipe.pipeline as EPL
    import echopipe.types as ET

    g = np.load(os.path.join(golden_dir, "chain.npz"))
    for name, ctx, data, grid, apod, interp in cases.chain_cases(ET):
        spec = EPL.bmode_chain(window=apod.window, f_number=apod.f_number,
                               interpolation=interp,
                               grid={"x_positions": grid.x_positions.tolist(),
                                     "z_positions": grid.z_positions.tolist()})
        spec["outputs"] = ["beamform", "dynamic_adjustment"]
        graph = EPL.build_graph(spec)
        # the registry entries are the B200 ones
        assert graph.nodes["beamform"].kind.factory.__module__.startswith("paper_1811_01566_b200")
        outs, timing = EPL.execute(graph, (ET.RfFrame(data), ctx))
        rf = _host(outs["beamform"].data if not hasattr(outs["beamform"], "numpy")
                   else outs["beamform"].numpy())
        disp = outs["dynamic_adjustment"].numpy()
        assert rf.tobytes() == g[f"{name}_rf"].tobytes(), name
        assert disp.dtype == g[f"{name}_disp"].dtype
        assert np.abs(disp - g[f"{name}_disp"]).max() <= 2e-5, name
        assert [n for n, _ in timing.stages] == ["beamform", "analytic_signal", "envelope",
                                                 "dynamic_adjustment"]


def test_echopipe_benchmark_stage_attribution(ep):
    """echopipe.benchmark over its own simulator with the B200 kinds: the
    per-stage host-clock times are each stage's own GPU work (the synchronous
    wrappers), so DAS dominates and the stages add up to the frame total."""
    import echopipe.environment as EE
    import echopipe.pipeline as EPL
    import echopipe.presets as EPR
    import echopipe.types as ET

    from paper_1811_01566_b200 import environment as ME

    ctx_m, grid_m, n_s = ME.config_geometry("cfg2")
    ctx = ET.AcquisitionContext(ctx_m.speed_of_sound, ctx_m.sampling_frequency,
                                ctx_m.n_elements, ctx_m.pitch,
                                ET.PwScheme(ctx_m.tx_scheme.angles_rad))
    spec = EPL.bmode_chain(grid={"x_positions": grid_m.x_positions.tolist(),
                                 "z_positions": grid_m.z_positions.tolist()})
    graph = EPL.build_graph(spec)
    env = EE.open_simulator(EPR.wire_phantom(), ctx, n_s, dtype=np.float32, seed=0,
                            noise_std=0.01)
    res = EPL.benchmark(graph, env, n_frames=6, warmup=2)
    st = dict(res.timing.stages)
    assert st["beamform"] > st["analytic_signal"] + st["envelope"] + st["dynamic_adjustment"]
    assert st["envelope"] > 0.0 and st["dynamic_adjustment"] > 0.0
    # the frame total is the sum of its stages plus Python overhead only
    for t in res.per_frame:
        assert sum(ms for _, ms in t.stages) <= t.total_ms + 1e-6
        assert t.total_ms - sum(ms for _, ms in t.stages) < 2.0
    # the reference's Table-1 grouping works on the B200 timings
    from paper_1811_01566_b200 import report as R

    rows = dict(R.stage_rows(graph, res))
    assert set(rows) == {"Beamforming", "Envelope Detection", "Dynamic Adjustment"}


def test_das_beamform_oracle_is_the_reference_oracle(golden_dir):
    """das_beamform_oracle (beamform.py:299-357) -- evaluated by the f64
    kernel -- gives the reference oracle's bits (f64 frames) and their f32
    cast (f32 frames) on the criterion-4 instances."""
    from paper_1811_01566_b200 import types as T

    g = np.load(os.path.join(golden_dir, "das_small.npz"))
    for i, (ctx, data, grid, apod) in enumerate(cases.criterion4_cases(T)):
        if i >= 12:
            break
        ref = g[f"{i}_f64_linear_oracle"]
        got = bm.das_beamform_oracle(bm.RfFrame(data), ctx, grid, apod, "linear").numpy()
        assert got.dtype == np.float64 and got.tobytes() == ref.tobytes(), i
        got32 = bm.das_beamform_oracle(bm.RfFrame(data.astype(np.float32)), ctx, grid, apod,
                                       "linear").numpy()
        ref32 = bm.das_beamform_oracle(bm.RfFrame(data.astype(np.float32).astype(np.float64)),
                                       ctx, grid, apod, "linear").numpy().astype(np.float32)
        assert got32.dtype == np.float32 and got32.tobytes() == ref32.tobytes(), i
