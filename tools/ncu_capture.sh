# ncu --set full of the pass_X and the TMA column passes of one 256^3 finite apply_K (tools/kbench.py),
# reduced on the box to CSV (raw metrics + per-source-line stalls) so gpurun_out stays small
mkdir -p gpurun_out/ncu
tag=${TAG:-r02}
timeout 600 ncu --set full --import-source on --clock-control none -k regex:x_pass_kernel --launch-skip 3 -c 1 -o /tmp/x256 -f python tools/kbench.py 256 3 ${KIN:-finite} > gpurun_out/ncu/x_$tag.log 2>&1; echo "ncu x rc=$?"
timeout 600 ncu --set full --import-source on --clock-control none -k regex:col_tma_kernel --launch-skip 8 -c 4 -o /tmp/col256 -f python tools/kbench.py 256 3 ${KIN:-finite} > gpurun_out/ncu/col_$tag.log 2>&1; echo "ncu col rc=$?"
for r in x256 col256; do
  ncu -i /tmp/$r.ncu-rep --page raw --csv > gpurun_out/ncu/${r}_${tag}_raw.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu/${r}_${tag}_sass.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page source --csv > gpurun_out/ncu/${r}_${tag}_src.csv 2>/dev/null
done
gzip -f gpurun_out/ncu/*_${tag}_*.csv
ls -la gpurun_out/ncu
