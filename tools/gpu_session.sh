timeout 300 python tools/kbench.py 256 20 finite
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "finite or c4_twin or p33 or svk or refresh" 2>&1 | grep -E "^E |passed|failed" | head -5
