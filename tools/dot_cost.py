"""Dev probe: cost of the fused p.Ap (DOT variant) of the headline operator
kernel -- CUDA events around back-to-back launches of the cp.async-staged
CG-form kernel without the dot (hexbp_apply_ring_deferred) and with it
(hexbp_cgd_apply_fused, which applies A to the workspace's unpadded p), on
the same random input."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_2109_05072_b200 as hx
from paper_2109_05072_b200 import _lib


class _View:  # zero-copy torch view of a raw device pointer
    def __init__(self, ptr, n):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<f8", "data": (ptr, False), "version": 3}


e = int(os.environ.get("E", "66"))
dims = (e, e, e)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh(dims, 7)))
ws = op.workspace()
ws.set_mode("fast")
L = _lib.lib()
n = op.size()
r_, p_, ap_ = C.c_void_p(), C.c_void_p(), C.c_void_p()
assert L.hexbp_workspace_vectors(ws._h, C.byref(r_), C.byref(p_), C.byref(ap_)) == 0
pv = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1)
torch.as_tensor(_View(p_.value, n), device="cuda").copy_(pv)
w = torch.empty_like(pv)
part = torch.zeros(4, dtype=torch.float64, device="cuda")
st = torch.cuda.current_stream()
sp = C.c_void_p(st.cuda_stream)


def nodot():
    assert L.hexbp_apply_ring_deferred(op._setup._h, ws._h, C.c_void_p(pv.data_ptr()), C.c_void_p(w.data_ptr()), 1,
                                       sp) == 0


def dot():
    assert L.hexbp_cgd_apply_fused(op._setup._h, ws._h, 1, C.c_void_p(part.data_ptr()), sp) == 0


for name, f in (("no dot", nodot), ("dot", dot)) * 6:
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(st)
    for _ in range(10):
        f()
    b.record(st)
    torch.cuda.synchronize()
    print(name, round(a.elapsed_time(b) / 10, 4), "ms")
