# Final GPU evidence of the session: tests, smoke, bench lines (the launch list / traffic stamp is
# re-captured separately whenever a hashed kernel source changes).
python -m pytest tests -m gpu -q 2>&1 | tail -2 > gpurun_out/final_gputest.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.txt 2>&1
python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err
python bench.py --impl reference > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err
python bench.py --dist --no-sweep --no-cpu-baseline > gpurun_out/final_bench_dist.json 2> gpurun_out/final_bench_dist.err
cat gpurun_out/final_gputest.txt gpurun_out/final_smoke.txt
