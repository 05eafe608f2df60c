set -x
L="paper_2109_05072_b200/build/variants/base/libhexbp_b200.so paper_2109_05072_b200/build/variants/split/libhexbp_b200.so"
python tools/ab_time.py $L > gpurun_out/ab3.txt 2>&1
python tools/ab_time.py paper_2109_05072_b200/build/variants/split/libhexbp_b200.so paper_2109_05072_b200/build/variants/base/libhexbp_b200.so >> gpurun_out/ab3.txt 2>&1
python tools/ab_time.py $L >> gpurun_out/ab3.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_fast_kernels.py tests/test_fast_scale.py tests/test_jacobi.py tests/test_harness.py tests/test_reference_kats.py tests/test_poisson.py -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
python tools/cg_timeline.py > gpurun_out/timeline_split.txt 2>&1
cat gpurun_out/ab3.txt
