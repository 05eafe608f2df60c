"""CUPTI timeline (torch.profiler) of the fast CG on the headline problem:
per-kernel durations and the idle gaps between consecutive kernels (dev tool)."""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile

import paper_2109_05072_b200 as hx

e = int(os.environ.get("E", "66"))
bp, p = int(os.environ.get("BP", "3")), int(os.environ.get("P", "7"))
dims = (e, e, e)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind(bp), hx.build_box_mesh(dims, p)))
A = hx.ConstrainedOperator(op) if bp != 1 else op
b = torch.from_numpy(hx.bench_rhs(bp, p, dims)).cuda()
x = torch.zeros_like(b)
hx.cg(A, b, x, 0.0, 5, mode=os.environ.get("MODE", "fast"))
x.zero_()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    hx.cg(A, b, x, 0.0, 20, mode=os.environ.get("MODE", "fast"))
    torch.cuda.synchronize()
evs = [ev for ev in prof.events() if ev.device_type.name == "CUDA"]
ks = sorted([(ev.time_range.start, ev.time_range.end, ev.name) for ev in evs], key=lambda t: t[0])
agg = {}
gaps = []
for i, (s, t, n) in enumerate(ks):
    k = n.replace("(anonymous namespace)::", "").split("(")[0][-60:]
    agg.setdefault(k, []).append(t - s)
    if i:
        gaps.append((s - ks[i - 1][1], ks[i - 1][2].split("(")[0][-30:] + f" #{i - 1}", k + f" #{i}"))
for i, (s_, t_, n_) in enumerate(ks[:8]):
    print(i, round((t_ - s_) / 1e3, 4), n_[:90])
for k, v in agg.items():
    print(f"{len(v):3d} x {sum(v) / len(v) / 1e3:8.4f} ms  {k}")
tot = (ks[-1][1] - ks[0][0]) / 1e3
busy = sum(t - s for s, t, _ in ks) / 1e3
print(f"span {tot:.3f} ms, busy {busy:.3f} ms, idle {tot - busy:.3f} ms over {len(ks)} kernels")
big = sorted(gaps, reverse=True)[:6]
for g in big:
    print(f"gap {g[0] / 1e3:.4f} ms after {g[1]} before {g[2]}")
