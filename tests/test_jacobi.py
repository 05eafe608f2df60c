"""Jacobi-preconditioned CG (solver.hpp:91-205).

CPU: the oracle's restatement of jacobi_diagonal / preconditioned cg against
the reference itself (oracle/_ref), bit for bit -- and the reference test
JacobiDiagonal.* semantics (test_solver.cpp:164-196).
GPU (-m gpu): the device diagonal and the device PCG against the oracle:
reference mode bit for bit (diagonal, iteration count, residual history),
fast mode within the fast-path tolerances.
"""
import os

import numpy as np
import pytest

import oracle
from oracle import Oracle, random_vector

HAVE_REF = os.path.exists(oracle.REF_SO)
CASES = [(1, 2, (2, 2, 2), 0.1), (3, 2, (2, 2, 2), 0.1), (5, 2, (2, 2, 2), 0.1), (3, 3, (3, 2, 4), 0.1),
         (5, 4, (2, 3, 2), 0.05), (1, 5, (2, 2, 1), 0.1), (3, 7, (2, 2, 2), 0.1), (3, 8, (1, 2, 2), 0.0)]


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (reference absent)")
@pytest.mark.parametrize("bp,p,dims,a", CASES)
def test_oracle_jacobi_diagonal_is_the_reference(bp, p, dims, a):
    o, r = Oracle(bp, p, dims, a), oracle.RefLib(bp, p, dims, a)
    for constrained in (0, 1):
        assert np.array_equal(o.jacobi_diagonal(constrained), r.jacobi_diagonal(constrained))


@pytest.mark.skipif(not HAVE_REF, reason="oracle/_ref not built (reference absent)")
@pytest.mark.parametrize("bp,p,dims,a", [(3, 2, (3, 3, 3), 0.1), (5, 3, (2, 3, 2), 0.1), (1, 2, (3, 2, 2), 0.1)])
def test_oracle_pcg_is_the_reference(bp, p, dims, a):
    o, r = Oracle(bp, p, dims, a), oracle.RefLib(bp, p, dims, a)
    b = o.bench_rhs()
    con = bp != 1
    d = r.jacobi_diagonal(con)
    ro = o.cg(b, rel_tol=1e-8, max_iter=500, constrained=con, diag=d)
    rr = r.cg(b, rel_tol=1e-8, max_iter=500, constrained=con, diag=d)
    assert ro["iterations"] == rr["iterations"]
    assert np.array_equal(ro["residual_history"], rr["residual_history"])
    assert np.array_equal(ro["x"], rr["x"])


def test_jacobi_semantics_oracle():
    """MassDiagonalPositive, PreconditioningDoesNotSlowCg (test_solver.cpp:175-196)."""
    assert (Oracle(1, 3, (3, 2, 1), 0.1).jacobi_diagonal(False) > 0).all()
    o = Oracle(3, 2, (3, 3, 3), 0.1)
    b = random_vector(14, o.n)
    bd = o.jacobi_diagonal(True)
    b[bd == 1.0] = 0.0  # boundary dofs (the constrained diagonal is 1 exactly there)
    plain = o.cg(b, rel_tol=1e-8, max_iter=2000)
    jac = o.cg(b, rel_tol=1e-8, max_iter=2000, diag=bd)
    assert plain["converged"] and jac["converged"]
    assert jac["iterations"] <= plain["iterations"]


# ---------------------------------------------------------------- GPU
def _op(bp, p, dims, a, mode):
    import paper_2109_05072_b200 as hx

    mesh = hx.build_box_mesh(dims, p, (1.0, 1.0, 1.0), a)
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), mesh))
    op.workspace().set_mode(mode)
    return hx, op


@pytest.mark.gpu
@pytest.mark.parametrize("bp,p,dims,a", CASES)
def test_device_jacobi_diagonal_bitwise(bp, p, dims, a):
    hx, op = _op(bp, p, dims, a, "reference")
    o = Oracle(bp, p, dims, a)
    assert np.array_equal(hx.jacobi_diagonal(op, device=False), o.jacobi_diagonal(False))
    assert np.array_equal(hx.jacobi_diagonal(hx.ConstrainedOperator(op), device=False), o.jacobi_diagonal(True))


@pytest.mark.gpu
@pytest.mark.parametrize("bp,p,dims,a", [(3, 3, (4, 3, 3), 0.1), (5, 2, (3, 3, 4), 0.1), (1, 4, (2, 3, 2), 0.1),
                                         (3, 7, (3, 3, 2), 0.1)])
def test_device_pcg_reference_mode_bitwise(bp, p, dims, a):
    hx, op = _op(bp, p, dims, a, "reference")
    o = Oracle(bp, p, dims, a)
    con = bp != 1
    A = hx.ConstrainedOperator(op) if con else op
    d = hx.jacobi_diagonal(A)
    b = hx.bench_rhs(bp, p, dims)
    x = np.zeros(op.size())
    rep = hx.cg(A, b, x, rel_tol=1e-8, max_iter=2000, diag=d)
    ref = o.cg(o.bench_rhs(), rel_tol=1e-8, max_iter=2000, constrained=con, diag=o.jacobi_diagonal(con))
    assert rep.iterations == ref["iterations"]
    assert np.array_equal(rep.residual_history, ref["residual_history"])
    assert np.array_equal(x, ref["x"])


@pytest.mark.gpu
@pytest.mark.parametrize("bp,p,dims,a", [(3, 3, (4, 3, 3), 0.1), (5, 2, (3, 3, 4), 0.1), (1, 4, (2, 3, 2), 0.1),
                                         (3, 7, (3, 3, 2), 0.1), (3, 7, (5, 4, 6), 0.1)])
def test_device_pcg_fast_mode(bp, p, dims, a):
    import torch

    hx, op = _op(bp, p, dims, a, "fast")
    o = Oracle(bp, p, dims, a)
    con = bp != 1
    A = hx.ConstrainedOperator(op) if con else op
    d = hx.jacobi_diagonal(A)
    b = torch.from_numpy(hx.bench_rhs(bp, p, dims)).cuda()
    x = torch.zeros_like(b)
    rep = hx.cg(A, b, x, rel_tol=1e-8, max_iter=2000, diag=d, mode="fast")
    ref = o.cg(o.bench_rhs(), rel_tol=1e-8, max_iter=2000, constrained=con, diag=o.jacobi_diagonal(con))
    assert rep.converged
    # north_star bar: same count, |d final| <= 1e-10 (profiles/r2_parity_fast.json)
    assert rep.iterations == ref["iterations"]
    assert abs(rep.final_rel_residual - ref["final_rel_residual"]) <= 1e-10
    assert np.linalg.norm(x.cpu().numpy() - ref["x"]) <= 1e-8 * np.linalg.norm(ref["x"])
    # plain CG afterwards on the same workspace is unaffected (preconditioner state cleared)
    x2 = torch.zeros_like(b)
    rep2 = hx.cg(A, b, x2, rel_tol=1e-8, max_iter=2000, mode="fast")
    # ... bit for bit the solve of a fresh workspace
    _, fresh = _op(bp, p, dims, a, "fast")
    x3 = torch.zeros_like(b)
    rep3 = hx.cg(hx.ConstrainedOperator(fresh) if con else fresh, b, x3, rel_tol=1e-8, max_iter=2000, mode="fast")
    assert rep2.iterations == rep3.iterations
    assert np.array_equal(rep2.residual_history, rep3.residual_history) and torch.equal(x2, x3)


@pytest.mark.gpu
def test_device_pcg_errors_and_semantics():
    hx, op = _op(3, 2, (3, 3, 3), 0.1, "reference")
    A = hx.ConstrainedOperator(op)
    d = hx.jacobi_diagonal(A, device=False)
    with pytest.raises(ValueError):
        hx.cg(A, np.zeros(op.size()), np.zeros(op.size()), diag=d[:-1])
    b = random_vector(14, op.size())
    b[d == 1.0] = 0.0
    x1, x2 = np.zeros(op.size()), np.zeros(op.size())
    plain = hx.cg(A, b, x1, rel_tol=1e-8)
    jac = hx.cg(A, b, x2, rel_tol=1e-8, diag=d)  # host diagonal accepted too
    assert plain.converged and jac.converged and jac.iterations <= plain.iterations
