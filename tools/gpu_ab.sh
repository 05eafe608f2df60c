python -m pytest tests/test_tma_staging.py tests/test_fast_kernels.py -x -q -m gpu 2>&1 | tail -2 > gpurun_out/gputest.txt
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
cat gpurun_out/gputest.txt; python -c "
import json;d=json.loads(open('gpurun_out/bench_full.json').read().strip().splitlines()[-1])
print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['roofline']['kernel_ms'], d['e2e']['value'])
for k in ['p_sweep','bp1_sweep_10M','bp5_p7_50M']:
    print(k, {p: round(v['roofline_frac'],3) for p,v in d[k].items()})
print({k: v['GDOFps'] for k,v in d['bp3_cg_to_1e-8_50M'].items()})
"
