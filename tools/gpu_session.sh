timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python tools/precond_variants.py > gpurun_out/precond_variants.jsonl 2> gpurun_out/precond_variants.err; tail -2 gpurun_out/precond_variants.err
