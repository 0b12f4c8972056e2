timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log
run() { echo "== $2" >> gpurun_out/stress.txt; timeout 300 python scripts/stress_plans.py --shape $1 --m $3 --reps 800 --requant --scheme $4 --cfgs "$2" 2>&1 | grep -v "^  mismatch" >> gpurun_out/stress.txt; }
run 11008x4096 auto 1 per-group
run 4096x11008 auto 16 per-channel
run 4096x4096 auto 128 per-group
run 4096x11008 auto 1024 per-group
cat gpurun_out/stress.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
