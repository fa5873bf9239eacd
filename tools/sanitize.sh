# compute-sanitizer over tools/sanitize_driver.py (one GPU). Logs into gpurun_out/sanitizer_*.log
mkdir -p gpurun_out
for tool in ${TOOLS:-memcheck racecheck synccheck initcheck}; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 17 --print-limit 50 \
    python tools/sanitize_driver.py > gpurun_out/sanitizer_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitizer_$tool.log
done
