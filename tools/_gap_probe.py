import ctypes as C, os, sys
sys.path.insert(0, os.getcwd())
import torch
from torch.profiler import ProfilerActivity, profile
import paper_2109_05072_b200 as hx
from paper_2109_05072_b200 import _lib
dims = (66, 66, 66)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh(dims, 7)))
ws = op.workspace(); ws.set_mode("fast")
L = _lib.lib(); n = op.size()
u = torch.rand(n, dtype=torch.float64, device="cuda"); w = torch.empty_like(u)
st = torch.cuda.current_stream()
def k():
    assert L.hexbp_apply_ring_deferred(op._setup._h, ws._h, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()), 1, C.c_void_p(st.cuda_stream)) == 0
k(); k(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    k(); k()
    w.zero_()
    k()
    x = torch.zeros(8, device="cuda"); x += 1
    k(); k()
    torch.cuda.synchronize()
ks = sorted([(e.time_range.start, e.time_range.end, e.name[:50]) for e in prof.events() if e.device_type.name == "CUDA"])
for i, (s, t, nm) in enumerate(ks):
    gap = (s - ks[i-1][1]) / 1e3 if i else 0
    print(f"{i} gap {gap:.4f} dur {(t - s) / 1e3:.4f} {nm}")
