timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_s7.json 2> gpurun_out/bench_s7.err; tail -1 gpurun_out/bench_s7.err
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | grep -E "^E |passed|failed" | head -8
