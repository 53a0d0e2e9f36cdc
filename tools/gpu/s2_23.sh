timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "^E |Error|FAILED|passed|failed" | head -20
