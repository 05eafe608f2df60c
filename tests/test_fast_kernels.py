"""Fast-mode element kernels at every (BP, p): the lane-split / multi-column
work decompositions of apply.cu (S lanes per pencil, KC element columns per
CTA) against the oracle (operator.hpp:396-414 restated in oracle/), on meshes
whose column count is not a multiple of any KC, plus the fused p.Ap of the CG
form (ring.cuh) against reference-mode CG on the same operator."""
import numpy as np
import pytest

import paper_2109_05072_b200 as hx
from oracle import Oracle, random_vector

TOL = 1e-12


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


@pytest.mark.gpu
@pytest.mark.parametrize("bp", [1, 3, 5])
@pytest.mark.parametrize("p", list(range(1, 9)))
def test_fast_apply_and_fused_dot(bp, p):
    dims = (5, 3, 4) if p <= 4 else (3, 5, 2)  # 15 columns: ragged for KC = 2, 3, 8
    o = Oracle(bp, p, dims, 0.02)
    mesh = hx.build_box_mesh(dims, p, (1.0, 1.0, 1.0), 0.02)
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), mesh))
    op.workspace().set_mode("fast")
    u = random_vector(77 + p, o.n)
    assert rel(op.apply(u), o.apply(u, False)) <= TOL
    assert rel(hx.ConstrainedOperator(op).apply(u), o.apply(u, True)) <= TOL
    A = hx.ConstrainedOperator(op) if bp != 1 else op
    b = hx.bench_rhs(bp, p, dims)
    xf, xr = np.zeros(op.size()), np.zeros(op.size())
    rf = hx.cg(A, b, xf, rel_tol=0.0, max_iter=8, mode="fast")
    rr = hx.cg(A, b, xr, rel_tol=0.0, max_iter=8, mode="reference")
    np.testing.assert_allclose(rf.residual_history, rr.residual_history, rtol=1e-9)
    assert rel(xf, xr) <= 1e-9


@pytest.mark.gpu
@pytest.mark.parametrize("bp,p", [(1, 1), (1, 3), (1, 8), (3, 4), (3, 8), (5, 5)])
def test_z_segmented_columns(bp, p):
    """Few columns, deep z: the kernel splits each column into z-segments
    that recompute the element below them (apply.cu z_segments); results and
    the fused CG dot must not change."""
    dims = (2, 3, 24)
    o = Oracle(bp, p, dims, 0.0)
    mesh = hx.build_box_mesh(dims, p)
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), mesh))
    op.workspace().set_mode("fast")
    u = random_vector(5 + p, o.n)
    w = op.apply(u)
    assert rel(w, o.apply(u, False)) <= TOL
    assert rel(hx.ConstrainedOperator(op).apply(u), o.apply(u, True)) <= TOL
    assert np.array_equal(op.apply(u), w)  # deterministic
    A = hx.ConstrainedOperator(op) if bp != 1 else op
    b = hx.bench_rhs(bp, p, dims)
    xf, xr = np.zeros(op.size()), np.zeros(op.size())
    rf = hx.cg(A, b, xf, rel_tol=0.0, max_iter=6, mode="fast")
    rr = hx.cg(A, b, xr, rel_tol=0.0, max_iter=6, mode="reference")
    np.testing.assert_allclose(rf.residual_history, rr.residual_history, rtol=1e-9)
