"""Manufactured-solution Poisson check on the GPU (
acceptance criterion 5, proj/tests/acceptance/acceptance_main.cpp:181-222):
u = sin(pi x) sin(pi y) sin(pi z), f = 3 pi^2 u on the unit cube, BP3 with the
box-boundary constraint, consistent load vector (assemble_load), Jacobi PCG
to 1e-8, discrete L2 error; the error ratios between 2, 4 and 8 elements
per direction must lie in [2^(p+0.5), 2^(p+1.5)].

Fixtures: the reference itself (tests/golden/make_golden_poisson.py over
oracle/_ref) -- load vectors, solutions, errors, iteration counts."""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "poisson.npz")


def gold():
    d = np.load(GOLD)
    return d, {(int(p), int(e)): (err, int(it)) for p, e, err, it in d["cases"]}


def test_golden_errors_converge_at_order_p_plus_1():
    """The reference's own errors satisfy its acceptance band (pins the fixture)."""
    _, cases = gold()
    for p in (1, 2, 3):
        e2, e4, e8 = (cases[(p, e)][0] for e in (2, 4, 8))
        lo, hi = 2.0 ** (p + 0.5), 2.0 ** (p + 1.5)
        assert lo <= e2 / e4 <= hi and lo <= e4 / e8 <= hi, (p, e2 / e4, e4 / e8)


def _f_and_exact():
    import torch

    pi = math.pi

    def exact(x, y, z):
        return torch.sin(pi * x) * torch.sin(pi * y) * torch.sin(pi * z)

    def rhs(x, y, z):
        return 3.0 * pi * pi * exact(x, y, z)

    return exact, rhs


@pytest.mark.gpu
@pytest.mark.parametrize("p", [1, 2, 3])
def test_poisson_convergence_on_gpu(p):
    import torch

    import paper_2109_05072_b200 as hx

    d, cases = gold()
    exact, rhs = _f_and_exact()
    errs = []
    for e in (2, 4, 8):
        mesh = hx.build_box_mesh((e, e, e), p)
        setup = hx.make_setup(hx.BPKind.BP3, mesh)
        mass = hx.make_setup(hx.BPKind.BP1, mesh)
        op = hx.OperatorHandle(hx.Backend.Cuda, setup)  # reference arithmetic (default mode)
        cop = hx.ConstrainedOperator(op)
        b = hx.assemble_load(mesh, setup, mass, rhs)
        b[hx.boundary_mask(mesh, setup)] = 0.0
        gb, gx = d[f"p{p}_e{e}_b"], d[f"p{p}_e{e}_x"]
        # the device load vector: the reference's up to libm-vs-CUDA sin ulps
        assert np.abs(b.cpu().numpy() - gb).max() <= 1e-13 * np.abs(gb).max()
        diag = hx.jacobi_diagonal(cop)
        # from the reference's own b the device PCG reproduces its solution bit for bit
        xg = torch.zeros_like(b)
        rep = hx.cg(cop, torch.from_numpy(gb).cuda(), xg, rel_tol=1e-8, max_iter=2000, diag=diag)
        assert rep.converged and rep.iterations == cases[(p, e)][1]
        assert np.array_equal(xg.cpu().numpy(), gx)
        # the full device pipeline
        x = torch.zeros_like(b)
        rep = hx.cg(cop, b, x, rel_tol=1e-8, max_iter=2000, diag=diag)
        assert rep.converged
        err = hx.discrete_l2_error(mesh, setup, mass, x, exact)
        assert abs(err - cases[(p, e)][0]) <= 1e-9 * cases[(p, e)][0], (err, cases[(p, e)][0])
        errs.append(err)
    lo, hi = 2.0 ** (p + 0.5), 2.0 ** (p + 1.5)
    assert lo <= errs[0] / errs[1] <= hi and lo <= errs[1] / errs[2] <= hi


@pytest.mark.gpu
@pytest.mark.parametrize("bp,p,dims,a", [(3, 2, (3, 2, 4), 0.1), (5, 3, (2, 3, 2), 0.05), (1, 1, (4, 3, 2), 0.0)])
def test_fe_helpers_match_the_reference(bp, p, dims, a):
    """node coordinates bitwise (mesh.hpp:107-119); interpolation round trip
    against a host restatement with the reference's basis and factors."""
    import torch

    import paper_2109_05072_b200 as hx
    from oracle import Oracle

    o = Oracle(bp, p, dims, a)
    mesh = hx.build_box_mesh(dims, p, (1.0, 1.0, 1.0), a)
    setup = hx.make_setup(hx.BPKind(bp), mesh)
    X = hx.node_coords(setup).cpu().numpy()
    assert np.array_equal(X.T.ravel(), o.coords().ravel())
    # interp of a linear function is exact at the mapped points: x_q = interp(x_nodes)
    xq = hx.quadrature_points(setup)
    u = torch.as_tensor(X[0] + 2.0 * X[1] - X[2], device="cuda")
    uq = hx.interp_to_qpts(setup, u)
    np.testing.assert_allclose(uq.cpu().numpy(), (xq[0] + 2.0 * xq[1] - xq[2]).cpu().numpy(), rtol=0, atol=1e-13)
    # transpose identity: <interp v, w>_q == <v, interp^T w>_L
    v = torch.rand(setup.l_size(), dtype=torch.float64, device="cuda")
    w = torch.rand(setup.num_elements(), setup.q ** 3, dtype=torch.float64, device="cuda")
    lhs = float((hx.interp_to_qpts(setup, v) * w).sum())
    rhs = float((v * hx.interp_transpose(setup, w)).sum())
    assert abs(lhs - rhs) <= 1e-12 * abs(lhs)
    # factors on the device == the reference AoS factors
    assert np.array_equal(hx.factors_device(setup).cpu().numpy().ravel(), o.factors())
