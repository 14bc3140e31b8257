timeout 300 python tools/kbench.py 512 5 small
timeout 1800 python tools/run_configs.py c5 --noprof > gpurun_out/c5.jsonl 2> gpurun_out/c5.err; tail -2 gpurun_out/c5.err; cat gpurun_out/c5.jsonl
