#!/bin/bash
# Round-end measurement on one B200: tests, smoke, contract bench, ncu evidence.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
if [ -z "$NOTEST" ]; then
  timeout 900 python -m pytest tests -m gpu -q --timeout 300 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
  timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  echo "smoke exit $?" >> gpurun_out/smoke.log
fi
if [ -z "$NOBENCH" ]; then
  timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
  echo "bench exit $?" >> gpurun_out/bench.err
fi
if [ -z "$NONCU" ]; then
  # launch list of the bench command (cold, serialised: compare shares)
  timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --quick > gpurun_out/ncu_bench.log 2>&1
  echo "ncu launch list exit $?" >> gpurun_out/ncu_bench.log
  # DRAM bytes of every GEMM of the bench step (-> scripts/traffic_summary.py -> profiles/rNN_traffic.json)
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:w4a8_gemm --csv --log-file gpurun_out/traffic.csv \
      python scripts/quick_bench.py --profile --ms 1,2,4,8,16,32,64,128,256,512,1024 > gpurun_out/traffic.log 2>&1
  # full captures of the dominant kernel at decode / mid / prefill M
  for spec in "4096x11008 1024" "4096x11008 128" "4096x11008 16" "4096x11008 1"; do
    set -- $spec
    timeout 300 ncu --set full --import-source on --clock-control none -k regex:w4a8_gemm -s 2 -c 1 \
        -o gpurun_out/prof_$1_m$2 -f python scripts/quick_bench.py --profile --shapes $1 --ms $2 > gpurun_out/ncu_$1_m$2.log 2>&1
  done
fi
tail -3 gpurun_out/pytest_gpu.log 2>/dev/null; tail -1 gpurun_out/smoke.log 2>/dev/null; tail -c 600 gpurun_out/bench.json; tail -3 gpurun_out/bench.err; tail -2 gpurun_out/ncu_bench.log
