set -x
for lib in base tf base tf; do
  echo "== $lib"
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 1 --ps 6,8 --dofs 1e7 --iters 20
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 5 --ps 7 --iters 20
done
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -2 gpurun_out/pytest_gpu.txt
