# z-segment sizing A/B on the small BP1 problems (HEXBP_SEG_WAVES / HEXBP_SEG_MIN, z_segments in apply.cu)
for cfg in "2 4" "3 4" "4 4" "4 3" "6 3" "2 4" "3 4" "4 3"; do
  set -- $cfg
  echo "== waves $1 min $2"
  HEXBP_SEG_WAVES=$1 HEXBP_SEG_MIN=$2 python tools/sweep_time.py --bp 1 --ps 5,6,7,8 --dofs 1e7 --iters 20
done
