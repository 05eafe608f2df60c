"""CPU-side checks of the product boundary: the C-ABI library loads and exports
every symbol include/hexbp_b200.h declares, host-only entry points behave,
and nothing silently falls back to the CPU when no GPU is present."""
import ctypes as C
import subprocess

import numpy as np
import pytest

import paper_2109_05072_b200 as hx
from paper_2109_05072_b200 import _lib


def test_library_exports_every_declared_symbol():
    syms = _lib.exported_symbols()
    assert len(syms) >= 19
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    missing = [s for s in syms if s not in exported]
    assert not missing, missing
    L = _lib.lib()
    for s in syms:
        assert getattr(L, s) is not None


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_bench_rhs_matches_oracle_recipe():
    from oracle import Oracle

    for bp, p, dims in [(3, 3, (5, 4, 3)), (1, 2, (9, 7, 5)), (5, 4, (2, 3, 4))]:
        o = Oracle(bp, p, dims, 0.0)
        ref = o.bench_rhs(20240101)
        assert np.array_equal(hx.bench_rhs(bp, p, dims), ref)
        assert np.array_equal(hx.bench_rhs(bp, p, dims, offset=17, count=40), ref[17:57])
    with pytest.raises(ValueError):
        hx.bench_rhs(3, 3, (2, 2, 2), offset=10**6, count=1)


def test_uniform_stream_is_the_verify_probe_stream():
    """hexbp_uniform_stream (the device verify's probe vectors) = mt19937_64 +
    uniform_real_distribution(-1, 1) as check_equivalence draws them
    (verify.hpp:64-70); pinned to the oracle's restatement of that stream."""
    from oracle import random_vector
    from paper_2109_05072_b200 import harness as H

    for seed, n in [(2024 ^ (3 << 32) ^ 125, 1000), (77, 17), (12345, 4096)]:
        assert np.array_equal(H._uniform_stream(seed, n), random_vector(seed, n))


def test_mesh_api_validation_mirrors_reference():
    with pytest.raises(ValueError, match="element counts"):
        hx.build_box_mesh((0, 1, 1), 2)
    with pytest.raises(ValueError, match="degree"):
        hx.build_box_mesh((1, 1, 1), 0)
    with pytest.raises(ValueError, match="amplitude"):
        hx.build_box_mesh((1, 1, 1), 2, deform_amplitude=0.2)
    m = hx.build_box_mesh((3, 2, 1), 2)
    assert m.num_nodes() == 7 * 5 * 3 and m.num_elements() == 6
    b = hx.boundary_nodes(m)
    from oracle import Oracle

    o = Oracle(3, 2, (3, 2, 1), 0.0)
    lib = o.lib
    lib.or_num_boundary.restype = C.c_int64
    lib.or_num_boundary.argtypes = [C.c_void_p]
    lib.or_boundary.argtypes = [C.c_void_p, C.POINTER(C.c_int32)]
    nb = lib.or_num_boundary(o.h)
    ref = np.zeros(nb, np.int32)
    lib.or_boundary(o.h, ref.ctypes.data_as(C.POINTER(C.c_int32)))
    assert np.array_equal(b, ref)
    assert hx.parse_bp("bp5") == hx.BPKind.BP5 and hx.to_string(hx.BPKind.BP3) == "bp3"
    assert hx.parse_backend("cuda") == hx.Backend.Cuda
    with pytest.raises(ValueError):
        hx.parse_backend("fused")
    assert hx.default_quad_points(hx.BPKind.BP3, 7) == 9 and hx.default_quad_points(hx.BPKind.BP5, 7) == 8


def test_no_cpu_fallback_without_gpu():
    if hx.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(hx.HexbpCudaError, match="no CPU fallback"):
        hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh((2, 2, 2), 3))


def test_invalid_setup_arguments():
    with pytest.raises(ValueError):
        hx.make_setup(hx.BPKind.BP3, hx.HexMesh((2, 2, 2), 11))  # degree > 10: no device path
