# A/B/C of the operator passes: several builds of libdbfft.so, interleaved, 2 repetitions (tools/kbench.py)
# AB_LIBS: space-separated .so paths; AB_CFGS: ';'-separated kbench argument lists
mkdir -p gpurun_out
IFS=';' read -ra CFGS <<< "${AB_CFGS:-256 20 finite;256 20 small}"
for rep in 1 2; do
for cfg in "${CFGS[@]}"; do
  for lib in ${AB_LIBS}; do
    echo "$(basename $lib) $cfg: $(DBFFT_LIB=$lib timeout 300 python tools/kbench.py $cfg 2>&1 | tail -1)"
  done
done; done
