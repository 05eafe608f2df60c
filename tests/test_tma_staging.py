"""TMA staging of the operator input (tma.cu): the single-GPU fast CG keeps its
vectors row-pitched and the DMMA kernels (BP3 / BP5, p = 7) stage each
element's 8^3 node block -- the gather of restriction.hpp:55-65 /
operator.hpp:223-225 -- with one TMA tensor copy. The staged values are the
same doubles the cp.async path loads, so the solve must be bitwise identical
to the same solve with the tensor copy switched off (HEXBP_NO_TMA_U=1: same
pitched vectors, cp.async staging; read once per process, so each side runs
in its own interpreter), on a mesh with an odd node-row length (Nx = 7 nx + 1
odd: the pitch pads one double per row) and one with an even one, multi-wave
and with a z march longer than the u ring."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2109_05072_b200 as hx
bp, dims = int(sys.argv[2]), tuple(int(v) for v in sys.argv[3].split(","))
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, 7, (1.0, 1.0, 1.0), 0.05)))
op.workspace().set_mode("fast")
b = hx.bench_rhs(bp, 7, dims)
x = np.zeros(op.size())
rep = hx.cg(hx.ConstrainedOperator(op), b, x, rel_tol=1e-10, max_iter=400, mode="fast")
print(json.dumps({"it": rep.iterations, "hist": list(rep.residual_history), "x": x.tobytes().hex()}))
"""


def solve(bp, dims, tma):
    env = dict(os.environ)
    env.pop("HEXBP_NO_TMA_U", None)
    if not tma:
        env["HEXBP_NO_TMA_U"] = "1"
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(bp), ",".join(map(str, dims))], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.gpu
@pytest.mark.parametrize("bp,dims", [(3, (6, 5, 9)), (3, (19, 17, 6)), (5, (7, 4, 10)), (5, (18, 17, 5))])
def test_tma_staged_cg_is_bitwise_the_cp_async_cg(bp, dims):
    a, b = solve(bp, dims, True), solve(bp, dims, False)
    assert a["it"] == b["it"] > 0
    assert a["hist"] == b["hist"]
    assert a["x"] == b["x"]


@pytest.mark.gpu
def test_tma_path_matches_oracle_cg():
    """The TMA-staged fast CG against the reference's CG (oracle) on the same problem."""
    sys.path.insert(0, ROOT)
    from oracle import Oracle

    dims = (5, 6, 7)
    a = solve(3, dims, True)
    o = Oracle(3, 7, dims, 0.05)
    b = np.asarray(__import__("paper_2109_05072_b200").bench_rhs(3, 7, dims))
    ref = o.cg(b, rel_tol=1e-10, max_iter=400)
    assert a["it"] == ref["iterations"]
    assert abs(a["hist"][-1] / a["hist"][0] - ref["final_rel_residual"]) <= 1e-10


@pytest.mark.gpu
@pytest.mark.parametrize("bp,dims", [(3, (9, 7, 6)), (5, (8, 9, 5))])
def test_cg_form_apply_on_the_pitched_direction_is_bitwise_the_plain_apply(bp, dims):
    """hexbp_apply_cg_form (u copied into the row-pitched search direction,
    TMA-staged kernel) against hexbp_apply_ring_deferred on the caller's
    unpadded vector (cp.async-staged kernel): same w on every node off the
    lateral ring (the ring-deferred form leaves a column partial on x-face
    nodes -- whichever neighbour column stores last -- and nothing on y-face
    rows; their values live in the lateral buffer)."""
    import ctypes as C

    import torch

    sys.path.insert(0, ROOT)
    import paper_2109_05072_b200 as hx
    from paper_2109_05072_b200 import _lib

    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, 7, (1.0, 1.0, 1.0), 0.05)))
    ws = op.workspace()
    ws.set_mode("fast")
    L = _lib.lib()
    g = torch.Generator().manual_seed(5)
    u = torch.rand(op.size(), generator=g, dtype=torch.float64).cuda() - 0.5
    w1, w2 = torch.zeros_like(u), torch.zeros_like(u)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    Nx, Ny = dims[0] * 7 + 1, dims[1] * 7 + 1
    idx = torch.arange(op.size(), device="cuda")
    off_ring = ((idx % Nx) % 7 != 0) & (((idx // Nx) % Ny) % 7 != 0)
    for con in (0, 1):
        w1.zero_()
        w2.zero_()
        assert L.hexbp_apply_ring_deferred(op._setup._h, ws._h, C.c_void_p(u.data_ptr()), C.c_void_p(w1.data_ptr()),
                                           con, st) == 0
        assert L.hexbp_apply_cg_form(op._setup._h, ws._h, C.c_void_p(u.data_ptr()), C.c_void_p(w2.data_ptr()), con,
                                     st) == 0
        torch.cuda.synchronize()
        assert torch.equal(w1[off_ring], w2[off_ring])
        assert w1[off_ring].abs().max().item() > 0
