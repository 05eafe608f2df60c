"""Where does the CG drift vs the reference come from? (runs on a GPU box)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2109_05072_b200 as hx
import oracle
from oracle import Oracle, random_vector

bp, p, dims, a = 3, 3, (12, 12, 12), 0.1
o = Oracle(bp, p, dims, a)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p, deform_amplitude=a)))
cop = hx.ConstrainedOperator(op)
for s in range(3):
    u = random_vector(100 + s, o.n)
    w = cop.apply(u)
    wr = o.apply(u, True)
    d = np.abs(w - wr) / np.abs(wr).max()
    print(f"apply rel err norm {np.linalg.norm(w - wr) / np.linalg.norm(wr):.3e}  max/elem {d.max():.3e}")
b = o.bench_rhs()
ref = o.cg(b, rel_tol=1e-8, max_iter=2000)
x = np.zeros(o.n)
gpu = hx.cg(cop, b, x, rel_tol=1e-8, max_iter=2000)
print("ref", ref["iterations"], ref["final_rel_residual"], "gpu", gpu.iterations, gpu.final_rel_residual)


def host_cg(apply, b, tol, maxit, dot):
    n = b.size
    x = np.zeros(n)
    r = b - apply(x)
    r0 = np.sqrt(dot(r, r))
    p_ = r.copy()
    rz = dot(r, r)
    hist = [r0]
    for k in range(1, maxit + 1):
        Ap = apply(p_)
        pAp = dot(p_, Ap)
        al = rz / pAp
        x += al * p_
        r -= al * Ap
        rn = np.sqrt(dot(r, r))
        hist.append(rn)
        if rn / r0 <= tol:
            break
        rzn = dot(r, r)
        be = rzn / rz
        rz = rzn
        p_ = r + be * p_
    return k, hist[-1] / r0


print("host CG, oracle apply, ref dot   :", host_cg(lambda v: o.apply(v, True), b, 1e-8, 2000, oracle.dot))
print("host CG, CUDA apply, ref dot     :", host_cg(lambda v: cop.apply(v), b, 1e-8, 2000, oracle.dot))
print("host CG, oracle apply, numpy dot :", host_cg(lambda v: o.apply(v, True), b, 1e-8, 2000, lambda a_, b_: float(a_ @ b_)))
rng = np.random.default_rng(0)
for eps in (2e-16, 1e-15, 4e-15):
    print(f"host CG, oracle apply*(1+{eps}U):", host_cg(lambda v: o.apply(v, True) * (1 + eps * rng.uniform(-1, 1, o.n)), b,
                                                  1e-8, 2000, oracle.dot))
