V=paper_2109_05072_b200/build/variants
for v in dotreg dotsm dotreg dotsm; do echo "== $v"; HEXBP_LIB=$V/$v/libhexbp_b200.so python tools/ctx_probe2.py 2>&1 | tail -4; done
for r in 1 2; do python tools/ab_time.py $V/dotreg/libhexbp_b200.so $V/dotsm/libhexbp_b200.so; done
