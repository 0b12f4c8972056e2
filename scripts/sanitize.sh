#!/bin/bash
# compute-sanitizer over one small case per tile plan / mode (scripts/sanitize_cases.py).
# Logs: gpurun_out/sanitizer_{memcheck,racecheck,synccheck,initcheck}.txt
mkdir -p gpurun_out
python scripts/sanitize_cases.py > gpurun_out/sanitizer_plain.txt 2>&1
echo "exit $?" >> gpurun_out/sanitizer_plain.txt
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool $extra --print-limit 50 \
      python scripts/sanitize_cases.py ${SAN_ARGS} > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$tool.txt
done
for f in gpurun_out/sanitizer_*.txt; do echo "== $f"; tail -4 $f; done
