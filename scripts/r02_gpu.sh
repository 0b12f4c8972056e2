#!/bin/bash
# Round-2 measurement call on one B200: GPU tests (+ the BASELINE §2 CPU sweep in
# the background), smoke, contract bench, TP plumbing check, decode timelines.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
REF_PID=""
if [ -n "$REFSWEEP" ]; then
  python scripts/ref_cpu_sweep.py > gpurun_out/ref_cpu_sweep.json 2> gpurun_out/ref_cpu_sweep.err &
  REF_PID=$!
fi
if [ -z "$NOTEST" ]; then
  timeout ${TEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke exit $?" >> gpurun_out/smoke.log
fi
[ -n "$REF_PID" ] && wait $REF_PID
if [ -z "$NOBENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS:---steps 20 --warmup 5} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench exit $?" >> gpurun_out/bench.err
fi
if [ -n "$TPCHECK" ]; then
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531 \
     bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo > gpurun_out/tp_gloo.json 2> gpurun_out/tp_gloo.err
  echo "tp exit $?" >> gpurun_out/tp_gloo.err
fi
if [ -n "$TIMELINE" ]; then
  for spec in $TIMELINE; do
    IFS=/ read shape m <<< "$spec"
    timeout 120 python scripts/timeline.py --shape $shape --m $m >> gpurun_out/timeline.txt 2>&1
    timeout 120 python scripts/timeline.py --shape $shape --m $m --pair >> gpurun_out/timeline.txt 2>&1
  done
fi
tail -15 gpurun_out/pytest_gpu.log 2>/dev/null; tail -1 gpurun_out/smoke.log 2>/dev/null; tail -c 400 gpurun_out/bench.json; tail -3 gpurun_out/bench.err; tail -c 300 gpurun_out/tp_gloo.json 2>/dev/null; tail -3 gpurun_out/tp_gloo.err 2>/dev/null
