timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "trace or c1 or c2_mixed or c4_twin" 2>&1 | grep -E "^E |passed|failed" | head -8
