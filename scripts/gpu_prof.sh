#!/bin/bash
# ncu captures of the GEMM kernel at decode / mid / prefill M plus a tile-plan sweep.
mkdir -p gpurun_out
SHAPE=${SHAPE:-4096x11008}
for M in ${MS:-16 128 1024}; do
  timeout 300 ncu --set full --import-source on --clock-control none -k regex:w4a8_gemm -s 2 -c 1 \
     -o gpurun_out/prof_${SHAPE}_m${M} -f python scripts/quick_bench.py --profile --shapes $SHAPE --ms $M \
     > gpurun_out/ncu_m${M}.log 2>&1
  echo "ncu M=$M exit $?" >> gpurun_out/ncu_m${M}.log
done
if [ -n "$SWEEP" ]; then
timeout 600 python scripts/quick_bench.py --shapes 4096x4096,4096x11008 --ms 16,128,1024 --fp16 \
  --cfgs 'auto;{"ntok":16,"split":1};{"ntok":16,"split":0};{"ntok":64,"split":1};{"ntok":128,"split":0};{"ntok":128,"split":1};{"ntok":256,"split":0};{"ntok":256,"split":1}' \
  > gpurun_out/sweep.log 2>&1
fi
tail -3 gpurun_out/ncu_m*.log; cat gpurun_out/sweep.log 2>/dev/null | tail -60
