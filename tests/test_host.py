"""CPU-only checks: the C-ABI library loads and exports every symbol declared
in include/bmode200.h (no compute without a GPU), the host-side contract
(types, errors, graph building) behaves like the reference's, and the
product path refuses to run without CUDA instead of falling back."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_1811_01566_b200 as bm
from paper_1811_01566_b200 import _native as N
from paper_1811_01566_b200 import build as B
from paper_1811_01566_b200.errors import (CycleDetected, DimensionMismatch, InvalidMetadata,
                                          NativeError, PortMismatch, UnknownOperator)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "bmode200.h")).read()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(bm_\w+)\(", src, re.M)))


def test_library_built_for_sm100a_and_exports_header_symbols():
    lib_path = B.build()
    lib = ctypes.CDLL(lib_path)
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(N.SIGNATURES), "ctypes signatures out of sync with the header"
    lib.bm_abi_version.restype = ctypes.c_int
    assert lib.bm_abi_version() == 4
    lib.bm_error_string.restype = ctypes.c_char_p
    assert lib.bm_error_string(4) == b"analytic signal needs axis length >= 2"


def test_library_contains_sm100a_code():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", B.LIB], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_geometry_struct_layout():
    # 16 int32 + 2 double + 10 pointers + rx_contig + tile_ls (int32), as a C
    # compiler lays out bm_das_geometry
    assert N.DasGeometry.rx_contig.offset == 16 * 4 + 2 * 8 + 10 * 8
    assert N.DasGeometry.tile_ls.offset == 16 * 4 + 2 * 8 + 10 * 8 + 4
    assert N.DasGeometry.rx_table.offset == 16 * 4 + 2 * 8 + 10 * 8 + 8
    assert N.DasGeometry.tx_ready.offset == 16 * 4 + 2 * 8 + 10 * 8 + 16
    assert N.DasGeometry.tx_ready_base.offset == 16 * 4 + 2 * 8 + 10 * 8 + 24
    assert N.DasGeometry.weight_pad.offset == 16 * 4 + 2 * 8 + 10 * 8 + 32
    assert N.DasGeometry.tile_ls_nearest.offset == 16 * 4 + 2 * 8 + 10 * 8 + 40
    assert ctypes.sizeof(N.DasGeometry) == 16 * 4 + 2 * 8 + 10 * 8 + 48


def test_debug_keys_match_header_enum():
    src = open(os.path.join(ROOT, "include", "bmode200.h")).read()
    enum = {k.lower(): int(v) for k, v in re.findall(r"BM_DBG_(\w+) = (\d+)", src)}
    count = enum.pop("count")
    assert enum == N.DEBUG_KEYS and count == len(enum)


def test_geometry_struct_matches_c_compiler(tmp_path):
    """offsetof / sizeof of bm_das_geometry as gcc lays it out == the ctypes mirror."""
    import shutil
    import subprocess

    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    fields = [f for f, _ in N.DasGeometry._fields_]
    src = tmp_path / "layout.c"
    src.write_text("#include <stdio.h>\n#include <stddef.h>\n#include \"bmode200.h\"\n"
                   "int main(void) {\n" +
                   "".join(f'  printf("%zu\\n", offsetof(bm_das_geometry, {f}));\n'
                           for f in fields) +
                   '  printf("%zu\\n", sizeof(bm_das_geometry));\n  return 0;\n}\n')
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [getattr(N.DasGeometry, f).offset for f in fields] + [ctypes.sizeof(N.DasGeometry)]
    assert got == want


def test_invalid_arguments_rejected_without_gpu():
    lib = N.load()
    g = N.DasGeometry()
    assert lib.bm_das_beamform(ctypes.byref(g), None, 0, None, 0, 1, None) == 1
    assert lib.bm_analytic_signal(0, None, None, 1, 8, 1, None, 0, None) == 1
    assert lib.bm_envelope_display(0, None, None, None, None, 1, 8, 4, 30.0, None, 0, None) == 1
    assert lib.bm_display(0, None, None, None, None, 1, 4, 30.0, None) == 1
    # host-frame upload: null / misaligned counter, decreasing piece ends,
    # a counter without values -- all refused before any CUDA call
    assert lib.bm_stream_write_u32(None, 1, None) == 1
    assert lib.bm_stream_write_u32(ctypes.c_void_p(2), 1, None) == 1
    buf = ctypes.create_string_buffer(64)
    p = ctypes.c_void_p(ctypes.addressof(buf))
    ends = (ctypes.c_int64 * 2)(32, 16)
    assert lib.bm_host_upload(p, p, p, ends, 2, None, None, None) == 1
    ends = (ctypes.c_int64 * 1)(16)
    assert lib.bm_host_upload(p, p, p, ends, 1, p, None, None) == 1
    assert lib.bm_host_upload(None, p, p, ends, 1, None, None, None) == 1
    assert lib.bm_host_upload(p, p, p, ends, 0, None, None, None) == 1
    assert lib.bm_display_tiles(0, None, 2, 9, 2, 4, None, None, 30.0, None) == 1
    assert lib.bm_pad_traces(0, None, 8, 1, 8, None, 8, None) == 1


def test_debug_overrides_roundtrip_without_gpu():
    """Tuning hooks are process-wide integers behind bm_debug_set/get (the
    library reads no environment variables); the context manager restores
    the previous value."""
    lib = N.load()
    assert lib.bm_debug_get(N.DEBUG_KEYS["das_ft"]) == 0
    with N.debug_overrides(das_ft=2, fft_path=3):
        assert lib.bm_debug_get(N.DEBUG_KEYS["das_ft"]) == 2
        assert lib.bm_debug_get(N.DEBUG_KEYS["fft_path"]) == 3
    assert lib.bm_debug_get(N.DEBUG_KEYS["das_ft"]) == 0
    assert lib.bm_debug_get(99) == 0 and lib.bm_debug_set(-1, 5) == 0
    src = "".join(open(p).read() for p in B.sources())
    assert "getenv" not in src


def test_no_cpu_fallback():
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    ctx = bm.AcquisitionContext(1540.0, 40e6, 4, 2e-4, bm.StaScheme((0, 1, 2, 3)))
    grid = bm.ImageGrid(np.linspace(-1e-3, 1e-3, 4), np.linspace(1e-3, 2e-3, 4))
    frame = bm.RfFrame(np.zeros((4, 4, 64), np.float32))
    with pytest.raises(NativeError):
        bm.das_beamform(frame, ctx, grid)
    with pytest.raises(NativeError):
        bm.analytic_signal(np.ones(8))


def test_types_mirror_reference_validation():
    with pytest.raises(InvalidMetadata):
        bm.RfFrame(np.array([[[np.nan]]]))
    with pytest.raises(DimensionMismatch):
        bm.RfFrame(np.zeros((2, 2)))
    with pytest.raises(InvalidMetadata):
        bm.PwScheme((2.0,))
    ctx = bm.AcquisitionContext(1540.0, 40e6, 8, 2e-4, bm.StaScheme(tuple(range(8))))
    with pytest.raises(InvalidMetadata):
        ctx.channel_elements(4)
    with pytest.raises(DimensionMismatch):
        bm.validate_pair(bm.RfFrame(np.zeros((3, 8, 16))), ctx)
    g = bm.default_grid(ctx, 256, "sta")
    assert g.shape == (256, 8)
    m = bm.centered_rx_map(128, 64, range(128))
    assert m.shape == (128, 64) and m.min() == 0 and m.max() == 127


def test_graph_building_like_reference():
    graph = bm.build_graph(bm.bmode_chain())
    assert graph.order == ["beamform", "analytic_signal", "envelope", "dynamic_adjustment"]
    spec = bm.bmode_chain()
    spec["nodes"][0]["kind"] = "warp"
    with pytest.raises(UnknownOperator):
        bm.build_graph(spec)
    spec = {"nodes": [{"name": "a", "kind": "identity"}, {"name": "b", "kind": "identity"},
                      {"name": "c", "kind": "identity"}],
            "edges": [{"from": "b", "to": "c"}, {"from": "c", "to": "b"}],
            "inputs": ["a"], "outputs": ["a"]}
    with pytest.raises(CycleDetected):
        bm.build_graph(spec)
    spec = bm.bmode_chain()
    spec["edges"].append({"from": "beamform", "to": "envelope"})
    with pytest.raises(PortMismatch):
        bm.build_graph(spec)


def test_register_into_foreign_registry():
    reg = {}
    kinds = bm.register_gpu_operators(registry=reg)
    assert sorted(reg) == ["analytic_signal", "beamform", "dynamic_adjustment", "envelope",
                           "fir_filter", "hk_estimator", "sliding_moments"]
    ports = {k.name: (k.input_kinds, k.output_kind) for k in kinds}
    assert ports["beamform"] == (("observation",), "rf_image")
    assert ports["fir_filter"] == (("observation",), "observation")  # pipeline.py:209
    assert ports["sliding_moments"] == (("envelope_image",), "moment_maps")  # :221-225
    assert ports["hk_estimator"] == (("envelope_image",), "hk_map")  # :226-228


def test_fir_spec_validation():
    """FirSpec mirrors sigproc.py:20-33: f64, read-only, EmptyCoefficients for
    empty or non-finite taps (test_sigproc.py:55-61)."""
    from paper_1811_01566_b200.errors import EmptyCoefficients

    spec = bm.FirSpec([1, 2, 3])
    assert spec.coefficients.dtype == np.float64 and not spec.coefficients.flags.writeable
    for bad in ([], [1.0, np.nan], [np.inf]):
        with pytest.raises(EmptyCoefficients):
            bm.FirSpec(bad)


def _sass_by_function():
    import subprocess

    out = subprocess.run(["cuobjdump", "-sass", B.build()], capture_output=True, text=True).stdout
    funcs, name = {}, None
    for line in out.splitlines():
        if "Function :" in line:
            name = line.split("Function :")[1].strip()
            funcs[name] = []
        elif name and "/*" in line:
            funcs[name].append(line)
    return funcs


def test_no_contracted_fma_in_das_kernels():
    """Bitwise parity needs every product rounded before it is added.  ptxas
    may contract f32x2 mul+add into FFMA2; the DAS kernels only allow FFMA2
    with a zero addend (a plain rounded product) and scalar FFMA only inside
    the correctly-rounded sqrt/div sequences."""
    funcs = _sass_by_function()
    das = {n: l for n, l in funcs.items() if "das_tma_kernel" in n}
    # (tma-32ch, tma-64ch, weighted tma-32ch, weighted tma-64ch) x {STA, PW}
    # x {nearest, linear} x {t0, no t0} x {identity map, general}
    # + 2 tma-128ch (uniform linear identity-map, STA | PW)
    # + 32 two-frames-per-pass tma (identity map) x {32, 64}ch x {uniform, weighted}
    # + 20 two-frames-per-thread tma (uniform identity map, no t0) x {STA, PW} x
    # {nearest, linear}: FP = 1 x {32, 64}ch, FP = 2 x {16, 32, 64}ch
    # + 16 four-frames-per-thread tma, same apertures, FP = 1 / 2 x {16, 32}ch
    # + 48 of them weighted, the weight mode compiled in (rectangular + F,
    #   Hann, Hann + F)
    # + 32 uniform four-frames-per-thread 16ch tma with a compile-time window
    #   (96 / 128 / 160 / 192 samples) x FP = 1 / 2 x {STA, PW} x {nearest, linear}
    # + 24 weighted FP = 2 ones with a 96-sample compile-time window, 16 / 32ch,
    #   with the weight mode compiled in (rectangular + F, Hann, Hann + F)
    # + 24 one-frame weighted ones (FP = FT = 1, 32 / 64ch, contiguous maps, no
    #   t0) with the weight mode compiled in
    assert len(das) == 262
    for n, lines in das.items():
        for l in lines:
            if "FFMA2" in l:
                assert "RZ" in l.split("FFMA2", 1)[1].split(";")[0], (n, l)
        # floor via the magic constant, rounding toward -inf, packed (FADD2)
        assert any("FADD2.RM" in l for l in lines), n
        # TMA window staging, mbarrier pipeline, delay table in tensor memory
        assert any("UTMALDG" in l for l in lines), n
        assert any("SYNCS" in l for l in lines), n
        assert any("LDTM" in l for l in lines) and any("STTM" in l for l in lines), n
