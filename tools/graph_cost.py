"""Dev probe: cost of the first (capturing) fixed-iteration solve vs later
replays on the headline problem, CUDA events per solve."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import torch

import paper_2109_05072_b200 as hx

dims = (66, 66, 66)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh(dims, 7)))
A = hx.ConstrainedOperator(op)
b = torch.from_numpy(hx.bench_rhs(3, 7, dims)).cuda()
x = torch.zeros_like(b)
hx.cg(A, b, x, 0.0, 3, mode="fast")
for it in range(4):
    x.zero_()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record()
    hx.cg(A, b, x, 0.0, 20, mode="fast")
    e1.record()
    torch.cuda.synchronize()
    print(f"solve {it}: {e0.elapsed_time(e1):.2f} ms device, {1e3 * (time.perf_counter() - h0):.2f} ms host")
