# Round-end measurement session on one B200 (logs under gpurun_out/): the default bench line, the
# ncu launch list of the same workload (cold, serialised: compare shares), ncu --set full of pass_X
# and the TMA column passes (tools/ncu_capture.sh), and per-pass kernel times of the other kinds.
mkdir -p gpurun_out
tag=${TAG:-r02}
timeout 900 python bench.py > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err; echo "bench rc=$?"
cut -c1-300 gpurun_out/bench_$tag.json
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_$tag.log 2>&1; echo "ncu launches rc=$?"
python tools/ncu_summary.py launches gpurun_out/launches_$tag.csv > gpurun_out/launch_shares_$tag.json; gzip -f gpurun_out/launches_$tag.csv
TAG=$tag bash tools/ncu_capture.sh
for c in "256 20 small" "512 5 j2" "128 40 finite"; do echo "$c: $(timeout 300 python tools/kbench.py $c 2>&1 | tail -1)"; done > gpurun_out/kbench_$tag.log
