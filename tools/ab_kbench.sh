# A/B of the operator passes: build/libdbfft_base.so vs the in-tree libdbfft.so (tools/kbench.py)
# AB_CFGS: ';'-separated kbench argument lists
mkdir -p gpurun_out
IFS=';' read -ra CFGS <<< "${AB_CFGS:-256 20 finite;256 20 small}"
for rep in 1 2; do
for cfg in "${CFGS[@]}"; do
  echo "base $cfg: $(DBFFT_LIB=build/libdbfft_base.so python tools/kbench.py $cfg 2>&1 | tail -1)"
  echo "new  $cfg: $(python tools/kbench.py $cfg 2>&1 | tail -1)"
done; done
