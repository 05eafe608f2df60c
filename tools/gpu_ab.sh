V=paper_2109_05072_b200/build/variants
HEXBP_LIB=$V/gg2/libhexbp_b200.so python -m pytest tests/test_fast_kernels.py -q -k "bp1 or 1-2 or 2-1" 2>&1 | tail -1
for r in 1 2; do for v in gg0 gg2; do echo "== $v"; HEXBP_LIB=$V/$v/libhexbp_b200.so BP=1 P=2 E=107 python tools/cg_timeline.py 2>/dev/null | grep "apply_kernel<2, 4, 0, 16, 2"; HEXBP_LIB=$V/$v/libhexbp_b200.so python -c "
import sys; sys.path.insert(0,'.')
import bench
print(bench.p_sweep(1, 10, 0, ps=(2,), dofs=10_000_000))"; done; done
