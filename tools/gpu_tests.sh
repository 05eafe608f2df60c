# GPU job: the full -m gpu suite (optionally a subset: $@)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 2400 python -m pytest ${@:-tests} -m gpu -q -x -rf > gpurun_out/pytest_gpu.txt 2>&1; tail -15 gpurun_out/pytest_gpu.txt
