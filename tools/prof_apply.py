"""Profiling driver: R operator applies (and optionally CG iterations) on one GPU.
    ncu --set full -k regex:bp_apply_kernel -s 3 -c 1 -o prof python tools/prof_apply.py --dims 66,66,66
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2109_05072_b200 as hx

ap = argparse.ArgumentParser()
ap.add_argument("--bp", type=int, default=3)
ap.add_argument("--p", type=int, default=7)
ap.add_argument("--dims", default="66,66,66")
ap.add_argument("--reps", type=int, default=6)
ap.add_argument("--cg", type=int, default=0)
ap.add_argument("--mode", default="fast")
a = ap.parse_args()
dims = tuple(int(x) for x in a.dims.split(","))
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(a.bp), hx.build_box_mesh(dims, a.p)))
op.workspace().set_mode(a.mode)
A = hx.ConstrainedOperator(op) if a.bp != 1 else op
u = torch.empty(op.size(), dtype=torch.float64, device="cuda").uniform_(-1, 1)
w = torch.empty_like(u)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(a.reps + 1)]
ev[0].record()
for i in range(a.reps):
    A.apply(u, w)
    ev[i + 1].record()
torch.cuda.synchronize()
print("apply ms:", [round(ev[i].elapsed_time(ev[i + 1]), 3) for i in range(a.reps)])
print("kernel:", op.workspace().kernel_info())
if a.cg:
    b = torch.from_numpy(hx.bench_rhs(a.bp, a.p, dims)).cuda()
    x = torch.zeros_like(b)
    rep = hx.cg(A, b, x, 0.0, a.cg, mode=a.mode)
    print("cg iters", rep.iterations)
