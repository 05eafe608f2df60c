V=paper_2109_05072_b200/build/variants
python -m pytest tests/test_fast_kernels.py -x -q -m gpu 2>&1 | tail -2
python tools/ab_sweep.py $V/nofill/libhexbp_b200.so $V/fill/libhexbp_b200.so $V/nofill/libhexbp_b200.so $V/fill/libhexbp_b200.so
