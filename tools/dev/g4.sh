for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r02_sanitizer_${tool}.log 2>&1; echo "$tool rc=$?"
  PCA_B200_MULTI_MAX_SITES=262144 timeout 900 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_cases.py > gpurun_out/r02_sanitizer_${tool}_multi.log 2>&1; echo "$tool multi rc=$?"
done
tail -3 gpurun_out/r02_sanitizer_*.log
