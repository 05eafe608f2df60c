set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
L="paper_2109_05072_b200/build/variants/base/libhexbp_b200.so paper_2109_05072_b200/build/variants/w12/libhexbp_b200.so paper_2109_05072_b200/build/variants/split/libhexbp_b200.so paper_2109_05072_b200/build/variants/o1/libhexbp_b200.so paper_2109_05072_b200/build/variants/w12split/libhexbp_b200.so paper_2109_05072_b200/build/variants/w12o1/libhexbp_b200.so"
python tools/ab_time.py $L > gpurun_out/ab2.txt 2>&1
python tools/ab_time.py $(echo $L | tr ' ' '\n' | tac) >> gpurun_out/ab2.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.txt 2>&1
tail -3 gpurun_out/pytest_gpu.txt
cat gpurun_out/ab2.txt
