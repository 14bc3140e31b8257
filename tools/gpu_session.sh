timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "svk or p33 or finite or c4_twin" 2>&1 | tail -5
