# late-trigger PDL build (DBF_PDL_LATE=1, DBFFT_PDL=1) vs the default build without PDL: bench steps back to back
mkdir -p gpurun_out
DBFFT_LIB=build/libdbfft_pdllate.so DBFFT_PDL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "solve or tma" > gpurun_out/pdl_late_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/pdl_late_tests.log
for v in base late base late; do
  if [ $v = late ]; then export DBFFT_LIB=build/libdbfft_pdllate.so DBFFT_PDL=1; else export DBFFT_LIB=build/libdbfft_base.so DBFFT_PDL=0; fi
  timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_pdl_$v.json 2>/dev/null
  python -c "
import json; d=json.load(open('gpurun_out/bench_pdl_$v.json')); print('$v', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['config']['pcg_loop']['pcg_loop'])"
done | tee gpurun_out/pdl_late_bench.log
