# compute-sanitizer over the device parity suite (golden hierarchies: every kernel family,
# cluster tail, last-CTA tickets, while-graph PCG)
mkdir -p gpurun_out/sanitizer
S=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 $S --tool $tool --target-processes all --print-limit 50 --log-file gpurun_out/sanitizer/$tool.log \
    python -m pytest tests/test_device_parity.py -x -q -p no:cacheprovider > gpurun_out/sanitizer/$tool.pytest.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitizer/summary.txt
  tail -2 gpurun_out/sanitizer/$tool.pytest.log >> gpurun_out/sanitizer/summary.txt
  grep -E "ERROR SUMMARY|RACECHECK SUMMARY|Error|error" gpurun_out/sanitizer/$tool.log | sort | uniq -c | sort -rn | head -8 >> gpurun_out/sanitizer/summary.txt
done
cat gpurun_out/sanitizer/summary.txt
