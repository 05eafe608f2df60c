"""GPU multipass backend (operator.hpp:318-394): the
five-pass pipeline on the device reproduces the reference's Multipass backend
bit for bit (golden fixtures from the reference itself,
tests/golden/make_golden_multipass.py), including the CG recurrence on it,
and agrees with the fused backend to the apply tolerance."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "multipass.npz")


def cases():
    d = np.load(GOLD)
    return [(i, int(c[0]), int(c[1]), (int(c[2]), int(c[3]), int(c[4])), float(c[5])) for i, c in enumerate(d["cases"])]


def test_parse_backend_and_fixture():
    import paper_2109_05072_b200 as hx

    assert hx.parse_backend("cuda-multipass") == hx.Backend.CudaMultipass
    assert len(cases()) == 8


@pytest.mark.gpu
@pytest.mark.parametrize("idx,bp,p,dims,a", cases())
def test_multipass_is_the_references_multipass(idx, bp, p, dims, a):
    import paper_2109_05072_b200 as hx

    d = np.load(GOLD)
    mesh = hx.build_box_mesh(dims, p, (1.0, 1.0, 1.0), a)
    setup = hx.make_setup(hx.BPKind(bp), mesh)
    mp = hx.OperatorHandle(hx.Backend.CudaMultipass, setup)
    u = d[f"c{idx}_u"]
    assert np.array_equal(mp.apply(u), d[f"c{idx}_w"])
    assert np.array_equal(hx.ConstrainedOperator(mp).apply(u), d[f"c{idx}_wc"])
    # CG on the multipass operator: the reference's recurrence bit for bit
    A = hx.ConstrainedOperator(mp) if bp != 1 else mp
    x = np.zeros(mp.size())
    rep = hx.cg(A, hx.bench_rhs(bp, p, dims), x, rel_tol=0.0, max_iter=12)
    assert np.array_equal(rep.residual_history, d[f"c{idx}_hist"])
    # fused backend agrees to the apply tolerance (BackendsAgreeWithOracle, test_operator.cpp:54-77)
    fu = hx.OperatorHandle(hx.Backend.Cuda, setup)
    wf = fu.apply(u)
    assert np.linalg.norm(wf - d[f"c{idx}_w"]) <= 1e-12 * np.linalg.norm(d[f"c{idx}_w"])


@pytest.mark.gpu
def test_multipass_rejects_fast_mode():
    import paper_2109_05072_b200 as hx

    op = hx.OperatorHandle(hx.Backend.CudaMultipass, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh((2, 2, 2), 2)))
    with pytest.raises(Exception):
        op.workspace().set_mode("fast")
