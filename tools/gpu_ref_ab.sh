set -x
for lib in base x2 x3 x4 base x2 x3 x4; do echo "== $lib"; HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/refmode_time.py 2>&1 | tail -1; done
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_jacobi.py tests/test_reference_kats.py tests/test_harness.py tests/test_multipass.py tests/test_fast_kernels.py tests/test_poisson.py -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
