#!/bin/bash
# A/B of developer library variants: quick sweep per variant (lib/<name>.so)
mkdir -p gpurun_out; rm -f gpurun_out/ab_*.log
for v in prod ${VARIANTS}; do
  if [ "$v" = "prod" ]; then L=""; else L="$PWD/paper_2406_09904_b200/lib/$v.so"; fi
  env ${L:+QQQ_LIB_PATH=$L} timeout 600 python scripts/quick_bench.py --shapes ${SHAPES:-4096x11008} --ms ${MS:-1,16,128,1024} ${QARGS} > gpurun_out/ab_$v.log 2>&1
  echo "== $v"; cat gpurun_out/ab_$v.log
done
for spec in ${TL}; do
  echo "== TL $spec" >> gpurun_out/ab_timeline.log
  QQQ_LIB_PATH=$PWD/paper_2406_09904_b200/lib/${TLLIB:-libqqq_b200_tl}.so timeout 120 python scripts/timeline.py $(echo $spec | tr ':' ' ') >> gpurun_out/ab_timeline.log 2>&1
done
