set -x
L="paper_2109_05072_b200/build/variants/tmpl/libhexbp_b200.so paper_2109_05072_b200/build/variants/zpre/libhexbp_b200.so"
python tools/ab_time.py $L > gpurun_out/ab5.txt 2>&1
python tools/ab_time.py paper_2109_05072_b200/build/variants/zpre/libhexbp_b200.so paper_2109_05072_b200/build/variants/tmpl/libhexbp_b200.so >> gpurun_out/ab5.txt 2>&1
python tools/ab_time.py $L >> gpurun_out/ab5.txt 2>&1
cat gpurun_out/ab5.txt
