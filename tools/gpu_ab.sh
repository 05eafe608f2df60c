V=paper_2109_05072_b200/build/variants
for r in 1 2; do for v in ru2 ru3 ru4 ru3m3; do echo "== $v"; HEXBP_LIB=$V/$v/libhexbp_b200.so python tools/cg_timeline.py 2>/dev/null | grep "ring_update_r_kernel<7, false"; done; done
