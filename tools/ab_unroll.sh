# WHILE-body unroll (DBFFT_LOOP_UNROLL) A/B: bench steps back to back on one box
mkdir -p gpurun_out
for u in 1 2 4 1 2 4; do
  DBFFT_LOOP_UNROLL=$u timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_unroll$u.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_unroll$u.json')); print('unroll=$u', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['config']['cg_iters_timed'])"
done | tee gpurun_out/unroll_bench.log
for u in 1 2 4; do echo "unroll=$u $(DBFFT_LOOP_UNROLL=$u timeout 600 python tools/run_configs.py c1 c2 c3 --noprof --warm 2>&1 | grep -o '"config": "c[0-9]"\|"ms_per_cg_iter_warm": [0-9.]*\|"cg_iters": [0-9]*' | tr '\n' ' ')"; done | tee gpurun_out/unroll_configs.log
