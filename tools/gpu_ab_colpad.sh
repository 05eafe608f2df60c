# A/B: u-staging pads + BP5 p = 2 stride override (colpad) against the previous build (prev)
for lib in prev colpad prev colpad; do
  echo "== $lib"
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 5 --ps 2,3,4,5 --iters 20
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 3 --ps 2,3 --iters 20
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 1 --ps 3,4,5 --dofs 1e7 --iters 20
done
