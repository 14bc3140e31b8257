timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E |FAILED|passed|failed" | head -8
timeout 600 python bench.py --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_s9.json 2> gpurun_out/bench_s9.err; tail -1 gpurun_out/bench_s9.err
