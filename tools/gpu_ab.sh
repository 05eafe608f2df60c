V=paper_2109_05072_b200/build/variants
python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/gputest.txt
python tools/ab_time.py $V/base/libhexbp_b200.so $V/tma/libhexbp_b200.so > gpurun_out/ab4.txt 2>&1
python tools/ab_time.py $V/tma/libhexbp_b200.so $V/base/libhexbp_b200.so >> gpurun_out/ab4.txt 2>&1
cat gpurun_out/gputest.txt gpurun_out/ab4.txt
