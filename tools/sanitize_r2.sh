# compute-sanitizer over every kernel (tools/sanitize_case.py); summaries -> gpurun_out/r2_sanitize_*.log
for tool in racecheck synccheck memcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_case.py c1 key stable shard \
    > gpurun_out/r2_sanitize_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/r2_sanitize_$tool.log
done
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_case.py c2 \
  > gpurun_out/r2_sanitize_memcheck_c2.log 2>&1; echo "exit $?" >> gpurun_out/r2_sanitize_memcheck_c2.log
