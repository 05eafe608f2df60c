V=paper_2109_05072_b200/build/variants
HEXBP_LIB=paper_2109_05072_b200/build/variants/gseg/libhexbp_b200.so python -m pytest tests/test_fast_scale.py tests/test_tma_staging.py -q 2>&1 | tail -1
for v in gone gseg gone gseg; do echo "== $v"; HEXBP_LIB=$V/$v/libhexbp_b200.so python tools/ctx_probe2.py 2>&1 | tail -2; HEXBP_LIB=$V/$v/libhexbp_b200.so python tools/ab_time.py $V/$v/libhexbp_b200.so | cut -c50-200; done
