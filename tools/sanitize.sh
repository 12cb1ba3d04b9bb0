#!/bin/bash
# compute-sanitizer over tools/sanitize_smoke.py; one summary line per tool
OUT=gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  PYTHONPATH=$PWD timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 --target-processes all python tools/sanitize_smoke.py \
     > $OUT/sanitize_$tool.log 2>&1
  echo "$tool exit=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize smoke ok' $OUT/sanitize_$tool.log | tr '\n' ' ')"
done
