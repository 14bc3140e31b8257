# compute-sanitizer memcheck / racecheck / synccheck over tools/sanitize_cases.py; summaries under
# gpurun_out/sanitize/ (tool, case, error summary line)
mkdir -p gpurun_out/sanitize
for tool in memcheck synccheck racecheck; do
  for c in ${CASES:-c1 finite16 j2_16 tma n512 loopback}; do
    extra=""
    [ $tool = racecheck ] && extra="--racecheck-report hazard"
    timeout ${TMO:-900} compute-sanitizer --tool $tool $extra --print-limit 20 python tools/sanitize_cases.py $c \
      > gpurun_out/sanitize/${tool}_$c.log 2>&1
    echo "$tool $c rc=$? : $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|case .* ok' gpurun_out/sanitize/${tool}_$c.log | tr '\n' ' ')"
  done
done
