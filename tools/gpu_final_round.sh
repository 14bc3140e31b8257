# Final measurement session of a round on one B200: bench line, ncu launch list, ncu --set full of
# pass_X and the column passes, kernel times of the other kinds (tools/gpu_profile_round.sh), then
# the whole-solve timings of c1..c5 (tools/run_configs.py, warm walks, no per-kernel profiler).
mkdir -p gpurun_out
TAG=${TAG:-r02final} bash tools/gpu_profile_round.sh
timeout 900 python tools/run_configs.py --noprof --warm > gpurun_out/configs_${TAG:-r02final}.jsonl 2> gpurun_out/configs_${TAG:-r02final}.err; echo "configs rc=$?"
tail -c 1500 gpurun_out/configs_${TAG:-r02final}.jsonl
