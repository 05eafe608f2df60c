python -m pytest tests -m gpu -q 2>&1 | grep -E "FAILED|^E |passed|failed" | head -20
