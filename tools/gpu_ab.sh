python -m pytest tests -m gpu -q 2>&1 | tail -1
L=paper_2109_05072_b200/libhexbp_b200.so
for r in 1 2; do for g in 0 1; do echo "graph=$g"; HEXBP_CG_GRAPH=$g python tools/ab_time.py $L | cut -c1-200; HEXBP_CG_GRAPH=$g python tools/ab_sweep.py $L | cut -c40-400; done; done
