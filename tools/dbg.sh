timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k config5 2>&1 | grep -E "error|passed|failed" | head -5
