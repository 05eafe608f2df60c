"""Argument guards of the Python mirror and the C ABI (the calls that would
otherwise write past a buffer): dtype / layout / device / length checks on
apply, cg and dot, and writes into non-contiguous or non-float64 host
outputs. Mirrors the reference's std::invalid_argument on length mismatch
(operator.hpp:268, solver.hpp:97)."""
import numpy as np
import pytest

import paper_2109_05072_b200 as hx
from oracle import Oracle, random_vector

pytestmark = pytest.mark.gpu


def _op(bp=3, p=2, dims=(2, 3, 2), a=0.1):
    return hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p, (1, 1, 1), a)))


def test_cg_rejects_wrong_dtype_device_x():
    import torch

    op = _op()
    n = op.size()
    b = torch.from_numpy(hx.bench_rhs(3, 2, (2, 3, 2))).cuda()
    with pytest.raises(ValueError):
        hx.cg(hx.ConstrainedOperator(op), b, torch.zeros(n, device="cuda"))  # float32
    with pytest.raises(ValueError):
        hx.cg(hx.ConstrainedOperator(op), b, torch.zeros(n, dtype=torch.float64))  # host tensor
    with pytest.raises(ValueError):
        hx.cg(hx.ConstrainedOperator(op), b, torch.zeros(2 * n, dtype=torch.float64, device="cuda")[::2])
    x = torch.zeros(n, dtype=torch.float64, device="cuda")
    rep = hx.cg(hx.ConstrainedOperator(op), b, x, rel_tol=1e-8, max_iter=200)
    assert rep.converged


def test_dot_rejects_mismatch_and_oversize():
    import torch

    op = _op()
    ws = op.workspace()
    n = op.size()
    a = torch.ones(n, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        ws.dot(a, torch.ones(n - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        ws.dot(a, torch.ones(n, dtype=torch.float32, device="cuda"))
    # the C ABI refuses lengths beyond the workspace's chunk-partial buffer
    # (2368 chunks of 4096 for a small setup)
    big = torch.ones(2368 * 4096 + 1, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        ws.dot(big, big)
    fits = big[:2368 * 4096]
    assert ws.dot(fits, fits) == float(fits.numel())
    assert ws.dot(a, a) == float(n)


def test_host_apply_into_foreign_outputs():
    op = _op()
    n = op.size()
    o = Oracle(3, 2, (2, 3, 2), 0.1)
    u = random_vector(3, n)
    ref = o.apply(u, constrained=False)
    w32 = np.zeros(n, np.float32)
    out = op.apply(u, w32)  # float32 output: computed in a fresh array, copied into w
    assert out.dtype == np.float64 and np.linalg.norm(out - ref) <= 1e-12 * np.linalg.norm(ref)
    assert np.allclose(w32, ref.astype(np.float32))
    buf = np.zeros(2 * n)
    view = buf[::2]  # strided view: never written through as if contiguous
    out = op.apply(u, view)
    assert np.array_equal(view, out) and np.all(buf[1::2] == 0.0)
    wrong = np.zeros(n + 1)
    out = op.apply(u, wrong)  # wrong size: a fresh array is returned, as the reference resizes
    assert out.size == n and np.all(wrong == 0.0)


def test_bc_values_are_accepted_and_ignored():
    """solver.hpp:60-65: the constrained apply copies u on the essential dofs;
    boundary_bcs(mesh, value) values are not used (the reference accepts any)."""
    mesh = hx.build_box_mesh((2, 3, 2), 2, (1, 1, 1), 0.1)
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, mesh))
    u = random_vector(4, op.size())
    w0 = hx.ConstrainedOperator(op).apply(u)
    for value in (0.0, 1.0, -3.5):
        assert np.array_equal(hx.ConstrainedOperator(op, hx.boundary_bcs(mesh, value)).apply(u), w0)


def _structured_table(dims, p):
    """mesh.hpp:74-82 numbering, restated with numpy for the check."""
    gx, gy = dims[0] * p + 1, dims[1] * p + 1
    n = np.arange(p + 1)
    out = []
    for ez in range(dims[2]):
        for ey in range(dims[1]):
            for ex in range(dims[0]):
                k, j, i = np.meshgrid(n, n, n, indexing="ij")
                out.append(((ex * p + i) + gx * ((ey * p + j) + gy * (ez * p + k))).ravel())
    return np.concatenate(out).astype(np.int32)


def test_reference_setup_restriction_is_validated(golden_equiv):
    idx, arr = golden_equiv
    case = next(c for c in idx if "error" not in c and c["bp"] == 3)
    k, dims, p = case["key"], case["dims"], case["p"]
    table = _structured_table(dims, p)
    s = hx.OperatorSetup.from_reference(3, p, dims, arr[k + "/B"], arr[k + "/D"], arr[k + "/G"], elem_to_global=table)
    bad = table.copy()
    bad[[1, 2]] = bad[[2, 1]]
    with pytest.raises(ValueError):
        s.check_restriction(bad)
    with pytest.raises(ValueError):
        s.check_restriction(table[:-1])
