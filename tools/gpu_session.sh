timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
timeout 900 python tools/run_configs.py c1 c2 c3 c4 p33 > gpurun_out/configs_s5.jsonl 2> gpurun_out/configs_s5.err; tail -2 gpurun_out/configs_s5.err
