python -m pytest tests/test_fast_scale.py -q 2>&1 | tail -3
