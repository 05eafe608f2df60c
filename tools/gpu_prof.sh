# GPU job: ncu of the headline kernel as the fast CG launches it (TMA-staged, CG form) + launch list of a short bench
set -x
M=sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on --kernel-name-base demangled -k "regex:bp3_p7_mma_kernel<\(bool\)1, \(bool\)1, \(bool\)1>" -s 2 -c 1 -o gpurun_out/r2s_mma_bp3_tma -f python tools/prof_apply.py --reps 0 --cg 6 > gpurun_out/ncu_tma.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2s_launches_bench.csv python bench.py --steps 3 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
python tools/cg_timeline.py > gpurun_out/r2s_cg_timeline.txt 2>&1
ls -la gpurun_out | tail -5
