timeout 900 python -m pytest tests -m gpu -x -q -k "j2 or c5" 2>&1 | grep -E "^E |FAILED|passed|failed" | head -5
timeout 900 python tools/run_configs.py c5 --incs 4 > gpurun_out/c5p2.jsonl 2> gpurun_out/c5p2.err; tail -1 gpurun_out/c5p2.err
