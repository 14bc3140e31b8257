# PDL on / off (DBFFT_PDL) back to back: whole solves (c1 c2 c3 c4, warm walks) and bench steps
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or tma" > gpurun_out/pdl_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pdl_tests.log
for rep in 1 2; do
for pdl in 0 1; do
  echo "PDL=$pdl $(DBFFT_PDL=$pdl timeout 600 python tools/run_configs.py c1 c2 c3 c4 --noprof --warm 2>&1 | tr '\n' ' ' | cut -c1-3000)"
done; done > gpurun_out/pdl_configs.log
for pdl in 0 1 0 1; do
  DBFFT_PDL=$pdl timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_pdl$pdl.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_pdl$pdl.json')); print('PDL=$pdl', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['config']['pcg_loop']['pcg_loop'])"
done > gpurun_out/pdl_bench.log
