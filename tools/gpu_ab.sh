V=paper_2109_05072_b200/build/variants
for r in 1 2; do for v in ex4 ex3 ex3g ex4g; do echo "== $v"; HEXBP_LIB=$V/$v/libhexbp_b200.so python tools/refmode_time.py 2>&1 | tail -1; done; done
