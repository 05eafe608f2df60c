set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_jacobi.py tests/test_reference_kats.py tests/test_harness.py tests/test_multipass.py -m gpu -q -x > gpurun_out/pytest_gpu.txt 2>&1; tail -3 gpurun_out/pytest_gpu.txt
python tools/refmode_time.py
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:blocked_reduce -c 12 --csv --log-file gpurun_out/reduce_launches.csv python tools/refmode_time.py > /dev/null 2>&1
python - <<'PY'
import csv
rows=list(csv.reader(open('gpurun_out/reduce_launches.csv')))
i=[k for k,r in enumerate(rows) if r and r[0]=='ID'][0]; h=rows[i]
for r in rows[i+1:]:
    if len(r)>5 and r[h.index('Metric Name')]=='gpu__time_duration.sum': print(r[h.index('Kernel Name')][:50], r[h.index('Metric Value')])
PY
