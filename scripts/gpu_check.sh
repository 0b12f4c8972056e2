#!/bin/bash
# One gpurun call: tests + smoke + optional quick sweep / bench. Output under gpurun_out/.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
if [ -z "$NOTEST" ]; then
timeout 1200 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/smoke.log
fi
if [ -n "$QUICK" ]; then
  timeout 600 python scripts/quick_bench.py $QUICK > gpurun_out/quick.log 2>&1
  echo "quick exit $?" >> gpurun_out/quick.log
fi
if [ -n "$BENCH" ]; then
  timeout 900 python bench.py $BENCH > gpurun_out/bench.log 2>&1
  echo "bench exit $?" >> gpurun_out/bench.log
fi
tail -25 gpurun_out/pytest_gpu.log 2>/dev/null; tail -2 gpurun_out/smoke.log 2>/dev/null; tail -30 gpurun_out/quick.log 2>/dev/null; tail -c 3000 gpurun_out/bench.log 2>/dev/null
