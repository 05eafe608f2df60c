"""Profiling driver (dev): R launches of the headline operator as the CG runs
it (hexbp_apply_cg_form; DOT=1 adds the fused p.Ap)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2109_05072_b200 as hx
from paper_2109_05072_b200 import _lib

dot = int(os.environ.get("DOT", "1"))
dims = (66, 66, 66)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh(dims, 7)))
ws = op.workspace()
ws.set_mode("fast")
L = _lib.lib()
u = torch.empty(op.size(), dtype=torch.float64, device="cuda").uniform_(-1, 1)
w = torch.empty_like(u)
sp = C.c_void_p(torch.cuda.current_stream().cuda_stream)
assert L.hexbp_apply_cg_form(op._setup._h, ws._h, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()), 1, sp) == 0
for _ in range(4):
    assert L.hexbp_apply_cg_form(op._setup._h, ws._h, None, C.c_void_p(w.data_ptr()), 1 | (2 * dot), sp) == 0
torch.cuda.synchronize()
