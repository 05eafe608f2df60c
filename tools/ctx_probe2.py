"""Dev probe: the headline operator as the CG launches it (TMA-staged, CG
form) with and without the fused p.Ap, alternating, CUDA events per launch."""
import ctypes as C
import os
import subprocess
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2109_05072_b200 as hx
from paper_2109_05072_b200 import _lib

dims = (66, 66, 66)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh(dims, 7)))
ws = op.workspace()
ws.set_mode("fast")
L = _lib.lib()
u = torch.empty(op.size(), dtype=torch.float64, device="cuda").uniform_(-1, 1)
w = torch.empty_like(u)
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)
assert L.hexbp_apply_cg_form(op._setup._h, ws._h, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()), 1, sp) == 0
for mode in (1, 3) * 6:
    ts = []
    for it in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        assert L.hexbp_apply_cg_form(op._setup._h, ws._h, None, C.c_void_p(w.data_ptr()), mode, sp) == 0
        e1.record(st)
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) for a, b in ts)
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip()
    print("dot" if mode & 2 else "no dot", "median", round(v[len(v) // 2], 4), "min", round(v[0], 4), "|", clk)
