"""Per-kernel durations of the fast CG iteration on the headline problem
(dev tool; run under ncu --cache-control none --clock-control none
--metrics gpu__time_duration.sum), plus CUDA-event time of the same solve."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2109_05072_b200 as hx

p, bp = int(os.environ.get("P", "7")), int(os.environ.get("BP", "3"))
e = int(os.environ.get("E", "66"))
dims = (e, e, e)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p)))
A = hx.ConstrainedOperator(op) if bp != 1 else op
b = torch.from_numpy(hx.bench_rhs(bp, p, dims)).cuda()
x = torch.zeros_like(b)
hx.cg(A, b, x, 0.0, 3, mode="fast")
ts = []
for rep in range(int(os.environ.get("REPS", "5"))):
    x.zero_()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    ev[0].record()
    hx.cg(A, b, x, 0.0, 20, mode="fast")
    ev[1].record()
    torch.cuda.synchronize()
    ts.append(ev[0].elapsed_time(ev[1]))
ts.sort()
print(f"K=20 min {ts[0]:.3f} median {ts[len(ts) // 2]:.3f} ms", flush=True)
