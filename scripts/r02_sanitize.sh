# compute-sanitizer over every kernel class (small shapes); logs under gpurun_out/
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_cases.py > gpurun_out/r02_san_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02_san_$tool.log
  tail -3 gpurun_out/r02_san_$tool.log
done
