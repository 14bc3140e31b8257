timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
timeout 1800 python tools/run_configs.py c5 --noprof > gpurun_out/c5b.jsonl 2> gpurun_out/c5b.err; tail -2 gpurun_out/c5b.err; cat gpurun_out/c5b.jsonl | cut -c1-400
