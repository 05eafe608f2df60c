# GPU job: BP1 p = 1, 2 thread-per-column sweep + ncu of the staged p = 2 kernel as the fast CG launches it
set -x
python tools/sk_sweep.py run > gpurun_out/r2t_sk4.jsonl 2>&1
HEXBP_LIB=paper_2109_05072_b200/build/variants/sk/libhexbp_b200.so HEXBP_SK_0_2=1000120 timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k "regex:tpc_mass" -s 2 -c 1 -o gpurun_out/r2t_bp1p2_tpc_stg -f python tools/prof_apply.py --bp 1 --p 2 --dims 107,107,107 --reps 0 --cg 4 > gpurun_out/ncu_bp1b.log 2>&1
