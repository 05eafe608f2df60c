for c in "1 2 107" "1 1 215" "1 8 26" "3 8 45" "3 2 183"; do set -- $c; echo "== BP$1 p=$2 E=$3"; BP=$1 P=$2 E=$3 python tools/cg_timeline.py 2>/dev/null | grep -E " x |span" | grep -v Mem; done > gpurun_out/tl_small.txt 2>&1
cat gpurun_out/tl_small.txt
