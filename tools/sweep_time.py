"""Per-p timing of the fast path: plain operator apply and fixed-iteration CG
(~50M DOFs per p), CUDA events on the current stream.
    python tools/sweep_time.py [--ps 2,3,4,5,6,7,8] [--bp 3] [--dofs 5e7]
"""
import argparse
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2109_05072_b200 as hx

ap = argparse.ArgumentParser()
ap.add_argument("--ps", default="2,3,4,5,6,7,8")
ap.add_argument("--bp", type=int, default=3)
ap.add_argument("--dofs", type=float, default=5e7)
ap.add_argument("--iters", type=int, default=10)
a = ap.parse_args()
for p in [int(x) for x in a.ps.split(",")]:
    e = 1
    while ((e + 1) * p + 1) ** 3 <= a.dofs:
        e += 1
    dims = (e, e, e)
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(a.bp), hx.build_box_mesh(dims, p)))
    op.workspace().set_mode("fast")
    A = hx.ConstrainedOperator(op) if a.bp != 1 else op
    n = op.size()
    u = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
    w = torch.empty_like(u)
    for _ in range(2):
        A.apply(u, w)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    torch.cuda.synchronize()
    ev[0].record()
    for _ in range(5):
        A.apply(u, w)
    ev[1].record()
    torch.cuda.synchronize()
    t_apply = ev[0].elapsed_time(ev[1]) / 5
    b = torch.from_numpy(hx.bench_rhs(a.bp, p, dims)).cuda()
    x = torch.zeros_like(b)
    hx.cg(A, b, x, 0.0, 2, mode="fast")
    x.zero_()
    torch.cuda.synchronize()
    ev[0].record()
    hx.cg(A, b, x, 0.0, a.iters, mode="fast")
    ev[1].record()
    torch.cuda.synchronize()
    t_cg = ev[0].elapsed_time(ev[1]) / a.iters
    print(f"p={p} dims={dims} n={n} apply_ms={t_apply:.3f} cg_ms_per_it={t_cg:.3f} GDOF/s={n / t_cg / 1e6:.2f}",
          flush=True)
    del op, A, u, w, b, x
    torch.cuda.empty_cache()
