mkdir -p gpurun_out
for tool in memcheck racecheck; do
  S2_FWD_2CTA=1 timeout 900 compute-sanitizer --tool $tool python tools/sanitize_run.py > gpurun_out/san_${tool}.log 2>&1
  echo "$tool rc=$?"; grep -E "ERROR SUMMARY|RACECHECK SUMMARY|ok$" gpurun_out/san_${tool}.log | tail -12
done
