"""Same-box A/B timing of library variants on the cfg3 problem (dev tool).
    python tools/ab_time.py lib1.so lib2.so ...   (each run in a fresh process)
Per library: the operator kernel in CG form (ring deferred, no dot), and a
fixed-iteration fast CG (ms per iteration), CUDA events, best of 3.
"""
import json
import os
import subprocess
import sys

CHILD = r'''
import ctypes as C, json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2109_05072_b200 as hx
from paper_2109_05072_b200 import _lib
dims = tuple(int(x) for x in os.environ.get("AB_DIMS", "66,66,66").split(","))
p = int(os.environ.get("AB_P", "7"))
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh(dims, p)))
ws = op.workspace(); ws.set_mode("fast")
L = _lib.lib(); n = op.size()
u = torch.empty(n, dtype=torch.float64, device="cuda").uniform_(-1, 1); w = torch.empty_like(u)
st = torch.cuda.current_stream()
def k():
    assert L.hexbp_apply_ring_deferred(op._setup._h, ws._h, C.c_void_p(u.data_ptr()), C.c_void_p(w.data_ptr()), 1, C.c_void_p(st.cuda_stream)) == 0
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
best_k = 1e9
for rep in range(3):
    for _ in range(2): k()
    torch.cuda.synchronize(); ev[0].record()
    for _ in range(10): k()
    ev[1].record(); torch.cuda.synchronize()
    best_k = min(best_k, ev[0].elapsed_time(ev[1]) / 10)
b = torch.from_numpy(hx.bench_rhs(3, p, dims)).cuda(); x = torch.zeros_like(b)
A = hx.ConstrainedOperator(op)
hx.cg(A, b, x, 0.0, 3, mode="fast")
best_cg = 1e9
for rep in range(3):
    x.zero_(); torch.cuda.synchronize(); ev[0].record()
    hx.cg(A, b, x, 0.0, 20, mode="fast")
    ev[1].record(); torch.cuda.synchronize()
    best_cg = min(best_cg, ev[0].elapsed_time(ev[1]) / 20)
# correctness of the variant: fast vs reference-mode apply on a multi-wave mesh
sm = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh((20, 18, 16), p, (1, 1, 1), 0.1)))
us = torch.empty(sm.size(), dtype=torch.float64, device="cuda").uniform_(-1, 1)
sm.workspace().set_mode("reference"); wr = hx.ConstrainedOperator(sm).apply(us)
sm.workspace().set_mode("fast"); wf = hx.ConstrainedOperator(sm).apply(us)
err = (torch.linalg.norm(wf - wr) / torch.linalg.norm(wr)).item()
print(json.dumps({"kernel_ms": best_k, "cg_ms_per_it": best_cg, "GDOFps": n / best_cg / 1e6, "rel_err": err}))
'''
for lib in sys.argv[1:]:
    env = dict(os.environ, HEXBP_LIB=os.path.abspath(lib))
    out = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
    line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]
    print(f"{lib}: {line}", flush=True)
