#!/bin/bash
# decode investigation: PC vs PG, stream-K vs whole tiles, timeline, ncu source page
mkdir -p gpurun_out
timeout 300 python scripts/quick_bench.py --shapes 4096x11008,4096x4096 --ms 1,16 --schemes per-channel,per-group \
  --cfgs 'auto;{"ntok":16,"split":1};{"ntok":16,"split":0}' > gpurun_out/inv_quick.log 2>&1
for spec in "--shape 4096x11008 --m 1" "--shape 4096x11008 --m 1 --scheme per-channel" "--shape 4096x11008 --m 1 --cfg {\"ntok\":16,\"split\":1}"; do
  echo "== $spec" >> gpurun_out/inv_timeline.log
  timeout 120 python scripts/timeline.py $spec >> gpurun_out/inv_timeline.log 2>&1
done
timeout 300 ncu --set full --import-source on --clock-control none -k regex:w4a8_gemm -s 2 -c 1 \
  -o gpurun_out/inv_m1 -f python scripts/quick_bench.py --profile --shapes 4096x11008 --ms 1 > gpurun_out/inv_ncu.log 2>&1
cat gpurun_out/inv_quick.log gpurun_out/inv_timeline.log; tail -3 gpurun_out/inv_ncu.log
