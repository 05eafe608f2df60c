set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/parity_fast.py > gpurun_out/parity_fast.json 2> gpurun_out/parity_fast.log
M=sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_tensor_subpipe_dmma.sum,sm__inst_executed_pipe_fp64.sum,sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --set full --metrics $M --clock-control none --import-source on -k regex:bp3_p7_mma -s 4 -c 1 -o gpurun_out/r2_mma_bp3 -f python tools/prof_apply.py --reps 2 --cg 6 > gpurun_out/ncu1.log 2>&1
timeout 600 ncu --set full --metrics $M --clock-control none --import-source on -k regex:bp5_p7_mma -s 4 -c 1 -o gpurun_out/r2_mma_bp5 -f python tools/prof_apply.py --bp 5 --dims 60,60,60 --reps 2 --cg 6 > gpurun_out/ncu2.log 2>&1
for p in 5 6 8; do
timeout 600 ncu --set full --metrics $M --clock-control none --import-source on -k regex:bp_apply_kernel -s 4 -c 1 -o gpurun_out/r2_dfma_bp3_p$p -f python tools/prof_apply.py --p $p --dims 40,40,40 --reps 2 --cg 6 > gpurun_out/ncu_p$p.log 2>&1
done
ls -la gpurun_out
