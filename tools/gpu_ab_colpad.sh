# A/B: BP3 p = 1 pencil-stride override (colpad) against the previous build (prev)
for lib in prev colpad prev colpad; do
  echo "== $lib"
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 3 --ps 1 --iters 20
done
