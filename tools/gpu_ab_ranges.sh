# A/B: DFMA element kernel before / after element-range support (pre / post variants)
for lib in pre post pre post; do
  echo "== $lib"
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 3 --ps 3,5,8 --iters 20
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 1 --ps 4,6,8 --dofs 1e7 --iters 20
done
