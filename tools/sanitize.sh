#!/bin/bash
# compute-sanitizer over tools/sanitize_cases.py (run under gpurun)
mkdir -p gpurun_out/sanitize
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 \
      python tools/sanitize_cases.py > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|SANITIZE CASES DONE' gpurun_out/sanitize/$tool.log | tr '\n' ' ')"
done
