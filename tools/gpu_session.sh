timeout 900 python tools/run_configs.py c1 c2 c3 p33 --noprof > gpurun_out/configs_g.jsonl 2>&1
DBFFT_GRAPHS=0 timeout 900 python tools/run_configs.py c1 c2 c3 p33 --noprof > gpurun_out/configs_ng.jsonl 2>&1
