"""Dev probe: fast CG on small problems (launch-bound regime), fixed
iterations, CUDA events, best of 5 -- for the HEXBP_CG_GRAPH A/B."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2109_05072_b200 as hx

for bp, p, e in ((3, 3, 33), (3, 7, 12), (1, 2, 40)):
    dims = (e, e, e)
    op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p)))
    A = hx.ConstrainedOperator(op) if bp != 1 else op
    b = torch.from_numpy(hx.bench_rhs(bp, p, dims)).cuda()
    x = torch.zeros_like(b)
    hx.cg(A, b, x, 0.0, 50, mode="fast")
    best = 1e9
    for _ in range(5):
        x.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        hx.cg(A, b, x, 0.0, 50, mode="fast")
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 50)
    print(f"bp{bp} p={p} {op.size()} DOFs: {best * 1e3:.1f} us/it, {op.size() / best / 1e6:.2f} GDOF/s")
