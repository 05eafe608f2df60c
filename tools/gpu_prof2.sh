# ncu of the reference-mode (bit-exact) operator and the weakest fast degrees
set -x
M=sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:bp_apply_exact -s 2 -c 1 -o gpurun_out/r2_exact_bp3_p7 -f python tools/prof_apply.py --reps 3 --mode reference > gpurun_out/ncu_exact.log 2>&1
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:bp_apply_kernel -s 4 -c 1 -o gpurun_out/r2_dfma_bp1_p2 -f python tools/prof_apply.py --bp 1 --p 2 --dims 107,107,107 --reps 2 --cg 6 > gpurun_out/ncu_bp1p2.log 2>&1
timeout 900 ncu --set full --metrics $M --clock-control none --import-source on -k regex:bp_apply_kernel -s 4 -c 1 -o gpurun_out/r2_dfma_bp5_p2 -f python tools/prof_apply.py --bp 5 --p 2 --dims 184,184,184 --reps 2 --cg 6 > gpurun_out/ncu_bp5p2.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 80 --csv --log-file gpurun_out/r2_launches_bp1p2.csv env BP=1 P=2 E=107 REPS=2 python tools/cg_breakdown.py > gpurun_out/bp1p2_breakdown.txt 2>&1
ls -la gpurun_out/*.ncu-rep
