python -m pytest tests/test_gpu_parity_r2.py -x -q -k "zsolve" 2>&1 | grep -E "Error|assert|FAILED|knobs|passed|failed" | head -20
python -m pytest tests -m gpu -x -q 2>&1 | tail -1
