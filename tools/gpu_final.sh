# Final GPU evidence of the session: tests, smoke, bench lines, launch list (traffic stamp).
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/final_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
cat gpurun_out/final_gputest.txt gpurun_out/final_smoke.txt
