# x += alpha p on a side stream beside F2 / F3 (DBFFT_XOVERLAP=k CTAs per SM) vs the default: tests, then bench steps back to back
mkdir -p gpurun_out
DBFFT_XOVERLAP=2 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_slab.py -m gpu -q -x -k "solve or c1 or c2 or newton or loopback or pcg" > gpurun_out/xoverlap_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/xoverlap_tests.log
for x in 0 1 2 0 1 2; do
  DBFFT_XOVERLAP=$x timeout 600 python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline > gpurun_out/bench_xo$x.json 2>gpurun_out/bench_xo$x.err || tail -3 gpurun_out/bench_xo$x.err
  python -c "
import json; d=json.load(open('gpurun_out/bench_xo$x.json')); k=d['kernel_ms']; n=d['roofline']['launches']
print('xoverlap=$x', d['value'], d['ms_per_step'], d['clocks']['sm_mhz'], d['config']['cg_iters_timed'], d['config']['pcg_loop']['pcg_loop'], {a: round(b/n,3) for a,b in k.items()})"
done | tee gpurun_out/xoverlap_bench.log
