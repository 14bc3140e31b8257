timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python tools/contrast_sweep.py 63 > gpurun_out/contrast63.jsonl 2> gpurun_out/contrast63.err; tail -2 gpurun_out/contrast63.err
