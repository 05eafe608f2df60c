import sys, os, torch
sys.path.insert(0, os.getcwd())
import paper_2109_05072_b200 as hx
dims=(66,66,66)
op = hx.OperatorHandle(hx.Backend.Cuda, hx.make_setup(hx.BPKind.BP3, hx.build_box_mesh(dims, 7)))
A = hx.ConstrainedOperator(op)
b = torch.from_numpy(hx.bench_rhs(3, 7, dims)).cuda(); x = torch.zeros_like(b)
hx.cg(A, b, x, 0.0, 3, mode="reference")
for rep in range(3):
    x.zero_(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); r = hx.cg(A, b, x, 0.0, 20, mode="reference"); e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1)/1e3
    print("reference-mode CG: %.3f ms/it, %.2f GDOF/s, final %.17g" % (t/20*1e3, op.size()*20/t/1e9, r.final_rel_residual))
