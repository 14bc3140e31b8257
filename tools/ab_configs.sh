# whole-solve A/B of two builds (DBFFT_LIB), back to back: c1 c2 c3 c4 warm walks
mkdir -p gpurun_out
for rep in 1 2; do
for lib in ${AB_LIBS}; do
  echo "$(basename $lib) $(DBFFT_LIB=$lib timeout 600 python tools/run_configs.py ${AB_CFGS:-c1 c2 c3 c4} --noprof --warm 2>/dev/null | python -c "
import sys, json
out = []
for ln in sys.stdin:
    try: d = json.loads(ln)
    except Exception: continue
    out.append('%s %.4f ms/it' % (d['config'], d['ms_per_cg_iter_warm']))
print('  '.join(out))")"
done; done
