"""The reference's operator / workspace / flop-counter unit tests
(proj/tests/unit/test_operator.cpp) restated for the device path."""
import json
import os
import threading

import numpy as np
import pytest

import paper_2109_05072_b200 as hx
from oracle import random_vector

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def op_for(bp, p, dims, a=0.0, backend=hx.Backend.Cuda, mode="reference", extent=(1.0, 1.0, 1.0)):
    op = hx.OperatorHandle(backend, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p, extent, a)))
    if backend == hx.Backend.Cuda:
        op.workspace().set_mode(mode)
    return op


BACKENDS = [(hx.Backend.Cuda, "reference"), (hx.Backend.Cuda, "fast"), (hx.Backend.CudaMultipass, "reference")]


@pytest.mark.parametrize("backend,mode", BACKENDS)
def test_mass_of_constant_integrates_volume(backend, mode):
    """test_operator.cpp:31-37"""
    op = op_for(1, 3, (1, 1, 1), backend=backend, mode=mode)
    w = op.apply(np.ones(op.size()))
    assert abs(w.sum() - 1.0) <= 1e-13


@pytest.mark.parametrize("backend,mode", BACKENDS)
@pytest.mark.parametrize("bp", [3, 5])
def test_stiffness_annihilates_constants(bp, backend, mode):
    """test_operator.cpp:39-52 (|A 1|_inf <= 1e-12 |A|_inf; max_i A_ii <= |A|_inf
    stands in for the assembled norm, a stricter bound)."""
    op = op_for(bp, 2, (2, 2, 2), 0.1, backend=backend, mode=mode)
    norm = np.abs(hx.jacobi_diagonal(op_for(bp, 2, (2, 2, 2), 0.1), device=False)).max()
    assert np.abs(op.apply(np.ones(op.size()))).max() <= 1e-12 * norm


@pytest.mark.parametrize("backend,mode", BACKENDS)
def test_galerkin_scaling_on_affine_element(backend, mode):
    """test_operator.cpp:164-175: one element on [0,h]^3 is the reference
    element's operator times h/2 (BP3); checked through applies."""
    h = 0.5
    a_ref = op_for(3, 2, (1, 1, 1), backend=backend, mode=mode, extent=(2.0, 2.0, 2.0))
    a_h = op_for(3, 2, (1, 1, 1), backend=backend, mode=mode, extent=(h, h, h))
    for seed in (1, 2, 3):
        u = random_vector(seed, a_ref.size())
        wr, wh = a_ref.apply(u), a_h.apply(u)
        assert np.abs(wh - wr * (h / 2.0)).max() <= 1e-12 * np.abs(wr).max() * (h / 2.0) * 8


def test_rejects_length_mismatch():
    """test_operator.cpp (RejectsLengthMismatch): std::invalid_argument."""
    op = op_for(1, 2, (1, 1, 1))
    with pytest.raises(ValueError):
        op.apply(np.zeros(op.size() + 1))


@pytest.mark.parametrize("mode", ["reference", "fast"])
def test_apply_allocates_nothing(mode):
    """test_operator.cpp (Workspace.FusedApplyAllocatesNothing): all device
    memory belongs to the setup / workspace; applies and CG allocate none."""
    import torch

    op = op_for(3, 3, (3, 3, 3), 0.1, mode=mode)
    u = torch.as_tensor(random_vector(71, op.size()), device="cuda")
    w = torch.empty_like(u)
    op.apply(u, w)
    torch.cuda.synchronize()
    free0 = torch.cuda.mem_get_info()[0]
    for _ in range(3):
        op.apply(u, w)
        hx.ConstrainedOperator(op).apply(u, w)
    hx.cg(hx.ConstrainedOperator(op), u, w, 0.0, 5, mode=mode)
    torch.cuda.synchronize()
    assert torch.cuda.mem_get_info()[0] == free0


def test_concurrent_applies_with_private_workspaces():
    """test_operator.cpp (Workspace.ConcurrentAppliesWithPrivateWorkspaces):
    two host threads, one workspace each, results bitwise equal to serial."""
    op = op_for(3, 2, (3, 2, 2), 0.1)
    u1, u2 = random_vector(81, op.size()), random_vector(82, op.size())
    ref1, ref2 = op.apply(u1), op.apply(u2)
    ws1, ws2 = op.make_workspace(), op.make_workspace()
    out = {}
    t1 = threading.Thread(target=lambda: out.__setitem__(1, op.apply(u1, ws=ws1)))
    t2 = threading.Thread(target=lambda: out.__setitem__(2, op.apply(u2, ws=ws2)))
    t1.start(), t2.start()
    t1.join(), t2.join()
    assert np.array_equal(out[1], ref1) and np.array_equal(out[2], ref2)


def test_flop_counter():
    """count_flops (operator.hpp:283-294) counts the CUDA kernel's own loops
    (an FMA = 1 mul + 1 add), so it tracks the reference's
    contract_dim trip counts (tests/golden/flops.json, per element) closely
    but not exactly; then the FlopCounter KATs of test_operator.cpp:236-272."""
    gold = json.load(open(os.path.join(HERE, "golden", "flops.json")))
    for key, v in gold.items():
        bp, p = int(key[2]), int(key.split("_p")[1])
        f = op_for(bp, p, (2, 2, 2)).count_flops()
        assert 0.8 <= (f.mul + f.add) / (v["mul"] + v["add"]) <= 1.25, (key, f, v)
        assert 0.9 <= f.mul / v["mul"] <= 1.1, (key, f, v)
    from paper_2109_05072_b200.harness import cost_model

    for p in range(1, 7):  # MatchesModelWithinQuarter
        f = op_for(5, p, (2, 2, 2)).count_flops()
        assert 0.75 < (f.mul + f.add) / cost_model(p, True)[0] < 1.25
    c3 = op_for(5, 3, (1, 1, 1)).count_flops()  # ScalesLikeFourthPower
    c7 = op_for(5, 7, (1, 1, 1)).count_flops()
    assert 11.0 < (c7.mul + c7.add) / (c3.mul + c3.add) < 17.0
    m = op_for(1, 2, (2, 2, 2)).count_flops()  # MassIsCheaperThanStiffness
    s = op_for(3, 2, (2, 2, 2)).count_flops()
    assert m.mul + m.add < s.mul + s.add
    fu = op_for(3, 3, (2, 2, 1), 0.1).count_flops()  # BackendsCountIdenticalElementWork
    mp = op_for(3, 3, (2, 2, 1), 0.1, backend=hx.Backend.CudaMultipass).count_flops()
    assert (fu.mul, fu.add) == (mp.mul, mp.add)


def test_multipass_owns_global_quadrature_fields():
    """test_operator.cpp (Workspace.MultipassOwnsGlobalQuadratureFields): the
    multipass workspace owns 2 x fields global quadrature fields, the fused
    one none. The fused path's element-level scratch is the ring-partial
    buffers that replace the E-vector (~4/p of the nodes plus per-plane
    corner copies): within one E-vector at p = 7, within two on tiny p = 3
    meshes."""
    for dims, p, bound in (((2, 2, 2), 3, 2.0), ((3, 3, 3), 7, 1.0)):
        mesh = hx.build_box_mesh(dims, p)
        for bp in (3, 5):
            setup = hx.make_setup(hx.BPKind(bp), mesh)
            mp = hx.OperatorHandle(hx.Backend.CudaMultipass, setup).workspace()
            fu = hx.OperatorHandle(hx.Backend.Cuda, setup).workspace()
            assert mp.qpoint_fields() >= 3 and fu.qpoint_fields() == 0
            evec_bytes = setup.num_elements() * (setup.p + 1) ** 3 * 8
            assert fu.global_bytes() <= bound * evec_bytes, (dims, p, fu.global_bytes(), evec_bytes)
            assert mp.global_bytes() >= 3 * 8 * setup.num_elements() * setup.q ** 3
