timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python tools/kbench.py 256 20 finite
timeout 300 python tools/kbench.py 256 10 small
