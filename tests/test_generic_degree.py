"""Generic degrees p = 9, 10 (the reference accepts any p, basis.hpp:86-111).
The fused kernels stop at p = 8 (the BASELINE range); a workspace of a p > 8
setup runs the multipass pipeline (multipass.cu) in reference arithmetic, so
its applies and CG recurrences are the reference's Multipass backend bit for
bit (golden fixtures from the reference itself,
tests/golden/make_golden_generic_p.py). CPU: the oracle restatement at these
degrees against the same fixtures."""
import os

import numpy as np
import pytest

from oracle import Oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden", "generic_p.npz")


def cases():
    d = np.load(GOLD)
    return [(i, int(c[0]), int(c[1]), (int(c[2]), int(c[3]), int(c[4])), float(c[5])) for i, c in enumerate(d["cases"])]


@pytest.mark.parametrize("idx,bp,p,dims,a", cases())
def test_oracle_generic_degree_is_the_reference(idx, bp, p, dims, a):
    d = np.load(GOLD)
    o = Oracle(bp, p, dims, a)
    u = d[f"c{idx}_u"]
    # the restatement follows the fused loop orders: bitwise against Backend::Fused,
    # apply tolerance against Backend::Multipass (BackendsAgreeWithOracle, test_operator.cpp:54-77)
    assert np.array_equal(o.apply(u), d[f"c{idx}_wf"])
    assert np.linalg.norm(o.apply(u) - d[f"c{idx}_w"]) <= 1e-12 * np.linalg.norm(d[f"c{idx}_w"])
    assert np.array_equal(o.jacobi_diagonal(False), d[f"c{idx}_diag"])
    assert np.array_equal(o.jacobi_diagonal(True), d[f"c{idx}_diagc"])


@pytest.mark.gpu
@pytest.mark.parametrize("idx,bp,p,dims,a", cases())
def test_generic_degree_device_is_the_references_multipass(idx, bp, p, dims, a):
    import paper_2109_05072_b200 as hx

    d = np.load(GOLD)
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p, (1.0, 1.0, 1.0), a)))
    u = d[f"c{idx}_u"]
    assert np.array_equal(op.apply(u), d[f"c{idx}_w"])
    assert np.array_equal(hx.ConstrainedOperator(op).apply(u), d[f"c{idx}_wc"])
    assert np.linalg.norm(op.apply(u) - d[f"c{idx}_wf"]) <= 1e-12 * np.linalg.norm(d[f"c{idx}_wf"])
    assert np.array_equal(hx.jacobi_diagonal(op, device=False), d[f"c{idx}_diag"])
    assert np.array_equal(hx.jacobi_diagonal(hx.ConstrainedOperator(op), device=False), d[f"c{idx}_diagc"])
    con = bp != 1
    A = hx.ConstrainedOperator(op) if con else op
    b = hx.bench_rhs(bp, p, dims)
    # "fast" requests run reference arithmetic at these degrees (api.cg)
    for mode in ("reference", "fast"):
        x = np.zeros(op.size())
        rep = hx.cg(A, b, x, rel_tol=0.0, max_iter=12, mode=mode)
        assert np.array_equal(rep.residual_history, d[f"c{idx}_hist"])
    x = np.zeros(op.size())
    rep = hx.cg(A, b, x, rel_tol=0.0, max_iter=12, diag=hx.jacobi_diagonal(A))
    assert np.array_equal(rep.residual_history, d[f"c{idx}_phist"])


@pytest.mark.gpu
def test_generic_degree_workspace_contract():
    import paper_2109_05072_b200 as hx

    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh((1, 1, 2), 9)))
    with pytest.raises(Exception, match="reference arithmetic only"):
        op.workspace().set_mode("fast")
    with pytest.raises(ValueError):
        hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh((1, 1, 1), 11))
