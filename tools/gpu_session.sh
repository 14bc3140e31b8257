PYTHONPATH=. timeout 300 python tools/dbg2.py
timeout 600 python bench.py > gpurun_out/bench_s11.json 2> gpurun_out/bench_s11.err; tail -3 gpurun_out/bench_s11.err
