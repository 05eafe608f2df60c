"""The headline (fast-mode) kernels at bench scale.

* The DMMA kernels (BP3 / BP5 p = 7) against the oracle on a multi-wave mesh:
  20 x 18 = 360 (BP3) / 24 x 20 = 480 (BP5) element columns (more than the
  2 / 3 x 148 resident CTAs, so the operator
  grid runs more than one wave and the last-CTA p.Ap ticket of ring.cuh is
  taken by a CTA of a later wave), 16 elements deep (the z march, the carried
  node plane and the 4-deep u staging ring run through many cycles).
* The fused p.Ap / ring-summing r-update of the fast CG on that mesh against
  the reference-arithmetic CG (same operator up to rounding).
* Fast vs reference-arithmetic operator at the headline configuration itself
  (BASELINE configs[2]: BP3 p = 7, 66^3 elements, 99.25M DOFs).
Tolerances: north_star's 1e-12 relative (verify.hpp:76-83) for the operator.
"""
import numpy as np
import pytest

import paper_2109_05072_b200 as hx
from oracle import Oracle, random_vector

pytestmark = pytest.mark.gpu
TOL = 1e-12


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def _op(bp, p, dims, a, mode):
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p, (1, 1, 1), a)))
    op.workspace().set_mode(mode)
    return op


# more element columns than resident CTAs (BP3: 2 per SM, BP5: 3 per SM)
DIMS = {3: (20, 18, 16), 5: (24, 20, 16)}


@pytest.mark.parametrize("bp", [3, 5])
def test_dmma_kernels_multiwave_against_oracle(bp):
    dims, a = DIMS[bp], 0.1
    o = Oracle(bp, 7, dims, a)
    op = _op(bp, 7, dims, a, "fast")
    assert op.size() == o.n
    info = op.workspace().kernel_info()
    assert dims[0] * dims[1] > info["ctas_per_sm"] * 148  # more than one wave of element columns
    for seed in (11, 12):
        u = random_vector(seed, o.n)
        assert rel(op.apply(u), o.apply(u, False)) <= TOL
        assert rel(hx.ConstrainedOperator(op).apply(u), o.apply(u, True)) <= TOL


@pytest.mark.parametrize("bp", [3, 5])
def test_fused_cg_multiwave_tracks_reference(bp):
    """p.Ap fused in the operator kernel (column partials + last-CTA finish),
    ring sums in the r-update: the first 12 iterates follow the
    reference-arithmetic solve to rounding."""
    import torch

    dims, a = DIMS[bp], 0.1
    opf, opr = _op(bp, 7, dims, a, "fast"), _op(bp, 7, dims, a, "reference")
    b = torch.from_numpy(hx.bench_rhs(bp, 7, dims)).cuda()
    xf, xr = torch.zeros_like(b), torch.zeros_like(b)
    rf = hx.cg(hx.ConstrainedOperator(opf), b, xf, rel_tol=0.0, max_iter=12, mode="fast")
    rr = hx.cg(hx.ConstrainedOperator(opr), b, xr, rel_tol=0.0, max_iter=12, mode="reference")
    assert rf.iterations == rr.iterations == 12
    np.testing.assert_allclose(rf.residual_history, rr.residual_history, rtol=1e-10)
    assert (torch.linalg.norm(xf - xr) / torch.linalg.norm(xr)).item() <= 1e-10
    # and run to run bitwise
    xf2 = torch.zeros_like(b)
    rf2 = hx.cg(hx.ConstrainedOperator(opf), b, xf2, rel_tol=0.0, max_iter=12, mode="fast")
    assert np.array_equal(rf.residual_history, rf2.residual_history) and torch.equal(xf, xf2)


def test_fast_vs_reference_operator_at_headline_config():
    """BASELINE configs[2] (cfg3): the DMMA kernel against the bit-exact
    reference-arithmetic kernel on the device, plain and constrained."""
    import torch

    dims = (66, 66, 66)
    op = _op(3, 7, dims, 0.0, "reference")
    assert op.size() == 99_252_847
    g = torch.Generator(device="cuda").manual_seed(5)
    u = torch.rand(op.size(), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    for con in (False, True):
        A = hx.ConstrainedOperator(op) if con else op
        op.workspace().set_mode("reference")
        wr = A.apply(u)
        op.workspace().set_mode("fast")
        wf = A.apply(u)
        err = (torch.linalg.norm(wf - wr) / torch.linalg.norm(wr)).item()
        assert err <= TOL, (con, err)
        del wr, wf


def test_fast_cg_at_headline_config_tracks_reference_mode():
    """The headline solve itself (cfg3, 20 fixed iterations as bench.py times
    it): the fast CG -- row-pitched vectors, TMA-staged DMMA operator, fused
    p.Ap and ring-summing r-update -- against the bit-exact reference-mode CG
    on the same device problem (the reference's own iterates)."""
    import torch

    dims = (66, 66, 66)
    op = _op(3, 7, dims, 0.0, "fast")
    A = hx.ConstrainedOperator(op)
    b = torch.from_numpy(hx.bench_rhs(3, 7, dims)).cuda()
    xf = torch.zeros_like(b)
    rf = hx.cg(A, b, xf, rel_tol=0.0, max_iter=20, mode="fast")
    op.workspace().set_mode("reference")
    xr = torch.zeros_like(b)
    rr = hx.cg(A, b, xr, rel_tol=0.0, max_iter=20, mode="reference")
    assert rf.iterations == rr.iterations == 20
    np.testing.assert_allclose(rf.residual_history, rr.residual_history, rtol=1e-10)
    assert abs(rf.final_rel_residual - rr.final_rel_residual) <= 1e-12
    assert (torch.linalg.norm(xf - xr) / torch.linalg.norm(xr)).item() <= 1e-10
