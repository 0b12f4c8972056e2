#!/bin/bash
# compute-sanitizer over one small case per tile plan / mode (scripts/sanitize_cases.py),
# on the sanitizer build (build.py -DQQQ_WATCHDOG_NS=600000000000ull -DQQQ_WATCHDOG_ITERS=0xffffffffu
# --name=san: the tools serialise CTAs, so the 4 s spin-wait watchdog of the product build would trap
# the stream-K owners). Logs: gpurun_out/sanitizer_{plain,memcheck,synccheck,racecheck,initcheck}.txt
mkdir -p gpurun_out
LIB=${SAN_LIB:-paper_2406_09904_b200/lib/san.so}
QQQ_LIB_PATH=$LIB python scripts/sanitize_cases.py > gpurun_out/sanitizer_plain.txt 2>&1
echo "exit $?" >> gpurun_out/sanitizer_plain.txt
for tool in memcheck synccheck racecheck initcheck; do
  extra=""
  [ "$tool" = racecheck ] && extra="--racecheck-report all"
  QQQ_LIB_PATH=$LIB timeout ${SAN_TIMEOUT:-1200} compute-sanitizer --tool $tool $extra --print-limit 50 \
      python scripts/sanitize_cases.py ${SAN_ARGS} > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "exit $?" >> gpurun_out/sanitizer_$tool.txt
done
for f in gpurun_out/sanitizer_*.txt; do echo "== $f"; tail -4 $f; done
