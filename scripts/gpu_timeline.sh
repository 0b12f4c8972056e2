#!/bin/bash
mkdir -p gpurun_out
for spec in "${@}"; do
  timeout 120 python scripts/timeline.py $spec >> gpurun_out/timeline.log 2>&1
done
cat gpurun_out/timeline.log
