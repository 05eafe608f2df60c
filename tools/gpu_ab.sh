V=paper_2109_05072_b200/build/variants
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/gputest.txt
for v in lbc tma; do echo "== $v"; HEXBP_LIB=$V/$v/libhexbp_b200.so python tools/cg_timeline.py 2>/dev/null | grep " x " | grep -v Mem; done > gpurun_out/tl.txt 2>&1
for r in 1 2; do python tools/ab_time.py $V/lbc/libhexbp_b200.so $V/tma/libhexbp_b200.so; done > gpurun_out/ab8.txt 2>&1
python bench.py --no-sweep --no-cpu-baseline > gpurun_out/bench_tma.json 2> gpurun_out/bench_tma.err
cat gpurun_out/gputest.txt gpurun_out/tl.txt gpurun_out/ab8.txt; python -c "
import json;d=json.loads(open('gpurun_out/bench_tma.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['kernel'])"
