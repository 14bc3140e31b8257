mkdir -p gpurun_out
for rep in 1 2; do
for lib in build/libdbfft_base.so build/libdbfft_p128.so build/libdbfft_pnone.so; do
  echo "$(basename $lib) 256 20 finite: $(DBFFT_LIB=$lib timeout 300 python tools/kbench.py 256 20 finite 2>&1 | tail -1)"
done
echo "kxpad 256 20 finite: $(DBFFT_KX_PAD=1 timeout 300 python tools/kbench.py 256 20 finite 2>&1 | tail -1)"
echo "kxpad 256 20 small: $(DBFFT_KX_PAD=1 timeout 300 python tools/kbench.py 256 20 small 2>&1 | tail -1)"
echo "base 256 20 small: $(timeout 300 python tools/kbench.py 256 20 small 2>&1 | tail -1)"
done
