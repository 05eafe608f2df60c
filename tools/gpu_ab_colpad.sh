# A/B: column padding of the DFMA element kernel's shared scratch (colpad / nocolpad variants)
for lib in nocolpad colpad nocolpad colpad; do
  echo "== $lib"
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 5 --ps 1,2,4,5 --iters 20
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 3 --ps 1,2,3 --iters 20
  HEXBP_LIB=paper_2109_05072_b200/build/variants/$lib/libhexbp_b200.so python tools/sweep_time.py --bp 1 --ps 3,4,8 --dofs 1e7 --iters 20
done
