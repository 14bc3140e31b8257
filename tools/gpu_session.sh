set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"col_tma|x_pass" -c 5 -o gpurun_out/full_s4 python tools/kbench.py 256 1 finite > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file gpurun_out/hist.csv -k regex:"k_phase_hist" python tools/kbench.py 256 1 finite > /dev/null 2>&1; grep -c hist gpurun_out/hist.csv
