"""Dev probe: the headline operator (CG form, TMA-staged) timed alone vs right
after a 2.4 GB streaming kernel (as in the CG, where it follows the x/p
update) -- CUDA events around the operator launch only."""
import ctypes as C
import os
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
n = op.size()
u = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
w = torch.empty_like(u)
a1, a2, a3 = (torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1) for _ in range(3))
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)
assert L.hexbp_apply_cg_form(op._setup._h, ws._h, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()), 1, sp) == 0


def opk():
    assert L.hexbp_apply_cg_form(op._setup._h, ws._h, None, C.c_void_p(w.data_ptr()), 1, sp) == 0


def stream_kernel():  # x/p-update-like: read 3 vectors, write 2
    a1.add_(a2, alpha=1e-3)
    a2.add_(a3, alpha=1e-3)


for mode in ("alone",) * 12 + ("after stream", "alone") * 3:
    ts = []
    for it in range(8):
        if mode != "alone":
            stream_kernel()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        opk()
        e1.record(st)
        ts.append((e0, e1))
    torch.cuda.synchronize()
    v = sorted(a.elapsed_time(b) for a, b in ts)
    import subprocess
    clk = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,power.draw,temperature.gpu,temperature.memory,clocks_event_reasons.active", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
    print(mode, "median", round(v[len(v) // 2], 4), "min", round(v[0], 4), "|", clk)
