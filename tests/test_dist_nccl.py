"""The library's multi-GPU path (hexbp_dist_*: NCCL communicator owned by the
library, boundary / interior split with the plane exchange overlapped, CG
scalars all-gathered) through its Python mirror parallel.NcclSlabOperator, on
the one GPU of the test box (world = 1: the overlap split, the carry combine
and the NCCL collectives all run; multi-rank halo sums are covered with the
same plane logic by tests/test_parallel_gloo.py and test_parallel_gpu.py)."""
import json
import os

import numpy as np
import pytest

import paper_2109_05072_b200 as hx
from paper_2109_05072_b200.parallel import NcclSlabOperator

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _single(bp, p, dims, a, mode="fast"):
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p, (1, 1, 1), a)))
    op.workspace().set_mode(mode)
    return op


@pytest.mark.parametrize("bp,p,dims", [(3, 7, (4, 3, 6)), (3, 7, (3, 4, 2)), (3, 7, (2, 2, 3)), (5, 7, (3, 3, 4)),
                                       (5, 7, (2, 3, 2)), (5, 4, (3, 3, 4)), (1, 3, (3, 2, 3)),
                                       # DFMA degrees (element ranges in apply.cu), z-segmented interior
                                       # ranges (BP3 p = 3: 3 columns per CTA, 8 interior layers), and the
                                       # thread-per-column BP1 p = 2 and BP5 p = 1 (no ranges: the unsplit launch)
                                       (3, 3, (2, 2, 10)), (3, 8, (2, 3, 3)), (3, 2, (4, 3, 5)), (5, 2, (2, 3, 4)),
                                       (5, 5, (2, 2, 4)), (1, 8, (2, 2, 3)), (1, 5, (3, 2, 6)), (1, 2, (3, 3, 3)),
                                       (5, 1, (3, 2, 4))])
@pytest.mark.parametrize("overlap", [True, False])
def test_distributed_apply_is_the_single_gpu_apply(bp, p, dims, overlap):
    """Bit for bit: the split launches assemble the inner planes with the same
    o(e) + carry(e-1) sums as the single launch's march."""
    import torch

    a = 0.1
    op = _single(bp, p, dims, a)
    dop = NcclSlabOperator(bp, p, dims, amplitude=a, overlap=overlap)
    assert dop.n_local == op.size()
    g = torch.Generator(device="cuda").manual_seed(9)
    u = torch.rand(op.size(), dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    for con in (False, True):
        w = (hx.ConstrainedOperator(op) if con else op).apply(u)
        wd = torch.empty_like(u)
        dop.apply(u, wd, con)
        torch.cuda.synchronize()
        assert torch.equal(w, wd), (con, (w - wd).abs().max().item())


@pytest.mark.parametrize("overlap", [True, False])
def test_distributed_cg_matches_reference_golden(overlap):
    """The fused distributed iteration on the golden bp3 p=7 6^3 a=0.1 case:
    the reference's 391 iterations and final residual within 1e-10."""
    import torch

    c = json.load(open(os.path.join(ROOT, "tests", "golden", "cg.json")))["bp3_p7_6_a0.1"]
    dop = NcclSlabOperator(3, 7, c["dims"], amplitude=c["a"], overlap=overlap)
    b = torch.from_numpy(hx.bench_rhs(3, 7, c["dims"])).cuda()
    x = torch.zeros_like(b)
    rep = dop.cg(b, x, rel_tol=1e-8, max_iter=2000, constrained=True)
    assert rep.iterations == c["iterations"] and rep.converged
    assert abs(rep.final_rel_residual - c["final_rel_residual"]) <= 1e-10
    assert abs(rep.residual_history[0] - c["residual_history"][0]) <= 1e-13 * c["residual_history"][0]
    # same solve on the single-GPU fast path
    xs = torch.zeros_like(b)
    rs = hx.cg(hx.ConstrainedOperator(_single(3, 7, c["dims"], c["a"])), b, xs, 1e-8, 2000, mode="fast")
    assert rs.iterations == rep.iterations
    assert (torch.linalg.norm(x - xs) / torch.linalg.norm(xs)).item() <= 1e-9


def test_distributed_cg_reference_mode():
    import torch

    c = json.load(open(os.path.join(ROOT, "tests", "golden", "cg.json")))["bp3_p3_12_a0.1"]
    dop = NcclSlabOperator(3, 3, c["dims"], amplitude=c["a"], mode="reference")
    b = torch.from_numpy(hx.bench_rhs(3, 3, c["dims"])).cuda()
    x = torch.zeros_like(b)
    rep = dop.cg(b, x, rel_tol=1e-8, max_iter=2000, constrained=True)
    assert rep.iterations == c["iterations"]
    assert abs(rep.final_rel_residual - c["final_rel_residual"]) <= 1e-10


def test_distributed_errors():
    with pytest.raises(ValueError):  # fewer element layers than ranks
        NcclSlabOperator(3, 2, (2, 2, 1), world=2, rank=0)


@pytest.mark.parametrize("overlap", [True, False])
def test_distributed_bp5_dmma_cg(overlap):
    """BP5 p = 7 (the DMMA kernel with the energy-form p.Ap, BASELINE configs[3]):
    the overlapped distributed solve against the single-GPU fast solve."""
    import torch

    dims, a = (4, 3, 5), 0.1
    dop = NcclSlabOperator(5, 7, dims, amplitude=a, overlap=overlap)
    b = torch.from_numpy(hx.bench_rhs(5, 7, dims)).cuda()
    x = torch.zeros_like(b)
    rep = dop.cg(b, x, rel_tol=1e-8, max_iter=3000, constrained=True)
    xs = torch.zeros_like(b)
    rs = hx.cg(hx.ConstrainedOperator(_single(5, 7, dims, a)), b, xs, 1e-8, 3000, mode="fast")
    assert rep.converged and abs(rep.iterations - rs.iterations) <= 1
    assert (torch.linalg.norm(x - xs) / torch.linalg.norm(xs)).item() <= 1e-8


@pytest.mark.parametrize("bp,p,dims", [(3, 4, (4, 3, 6)), (1, 6, (3, 3, 4))])
def test_distributed_dfma_cg(bp, p, dims):
    """A DFMA degree's overlapped distributed solve (boundary / interior
    element ranges) against the single-GPU fast solve."""
    import torch

    a = 0.1
    con = bp != 1
    dop = NcclSlabOperator(bp, p, dims, amplitude=a, overlap=True)
    b = torch.from_numpy(hx.bench_rhs(bp, p, dims)).cuda()
    x = torch.zeros_like(b)
    rep = dop.cg(b, x, rel_tol=1e-8, max_iter=3000, constrained=con)
    xs = torch.zeros_like(b)
    op = _single(bp, p, dims, a)
    rs = hx.cg(hx.ConstrainedOperator(op) if con else op, b, xs, 1e-8, 3000, mode="fast")
    assert rep.converged and abs(rep.iterations - rs.iterations) <= 1
    assert (torch.linalg.norm(x - xs) / torch.linalg.norm(xs)).item() <= 1e-8
