python -m pytest tests -m gpu -q -x 2>&1 | grep -E "FAILED|^E |passed|failed" | head -20
python -c "
import sys; sys.path.insert(0,'.')
import bench
print(bench.p_sweep(3, 10, 0, ps=(5, 6, 8)))
"
