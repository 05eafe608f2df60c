# generic GPU job: full GPU tests, fast-mode parity record, default bench line
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
python tools/parity_fast.py > gpurun_out/parity_fast.json 2> gpurun_out/parity_fast.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log; tail -c 3000 gpurun_out/bench.json
