#!/bin/bash
# usage: runbench.sh tag [extra args]
tag=$1; shift
python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline "$@" > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
tail -2 gpurun_out/bench_$tag.err
python -c "
import json
d=json.load(open('gpurun_out/bench_$tag.json')); r=d['roofline']; a=r['apply_K']
print('$tag value=%.3e ms/step=%.1f X=%.3f ms frac=%.3f applyK=%.3f ms frac=%.3f survey=%.3f' % (d['value'], d['ms_per_step'], r['avg_launch_ms'], r['frac'], a['avg_ms'], a['frac'], a['frac_of_survey_model']))
n=r['launches']; print({k: round(v/n,3) for k,v in d['kernel_ms'].items()})
"
