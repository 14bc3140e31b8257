set -x
timeout 600 python bench.py > gpurun_out/bench_s12.json 2> gpurun_out/bench_s12.err; tail -1 gpurun_out/bench_s12.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_s12_ref.json 2> gpurun_out/bench_s12_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_s12.csv python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; tail -1 gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none -k regex:"col_tma|x_pass|k_cg_direction" --launch-skip 44 -c 3 -o gpurun_out/full_s12 python bench.py --steps 1 --warmup 0 --e2e-steps 0 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; tail -1 gpurun_out/ncu_full.log
ls -la gpurun_out
