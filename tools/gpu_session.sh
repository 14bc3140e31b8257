timeout 300 python tools/kbench.py 512 5 small | python -c "import json,sys; d=json.load(sys.stdin); print(d['apply_ms'], d['passes']['pass_X'])"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "tma or c5 or j2" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
