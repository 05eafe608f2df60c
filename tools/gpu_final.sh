# Final GPU evidence of the session: tests, smoke, bench lines, launch list, ncu of the headline kernel.
set -x
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/final_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --dist --no-sweep --no-cpu-baseline > gpurun_out/final_bench_dist.json 2> gpurun_out/final_bench_dist.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
M=sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on --kernel-name-base demangled -k "regex:bp3_p7_mma_kernel<\(bool\)1, \(bool\)1, \(bool\)1>" -s 2 -c 1 -o gpurun_out/r2s_mma_bp3_final -f python tools/prof_apply.py --reps 0 --cg 6 > gpurun_out/ncu_final.log 2>&1
python tools/cg_timeline.py > gpurun_out/r2s_cg_timeline.txt 2>&1
cat gpurun_out/final_gputest.txt gpurun_out/final_smoke.txt
