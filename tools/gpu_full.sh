# GPU job: full test suite, smoke, default bench line (+ reference arm)
set -x
lscpu | head -20
timeout 2400 python -m pytest tests -m gpu -q -x -rf > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.log; tail -c 1500 gpurun_out/bench.json
python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; cat gpurun_out/bench_ref.json
