timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
python tools/cg_timeline.py > gpurun_out/r2s_cg_timeline.txt 2>&1
ls -la gpurun_out/r2s_launches_bench.csv
