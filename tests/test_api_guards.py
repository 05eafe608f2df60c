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
