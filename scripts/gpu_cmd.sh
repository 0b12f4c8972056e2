run() { echo "== $2" >> gpurun_out/stress.txt; timeout 300 python scripts/stress_plans.py --shape $1 --m $3 --reps 800 --requant --scheme $4 --cfgs "$2" 2>&1 | grep -v "^  mismatch" >> gpurun_out/stress.txt; }
run 11008x4096 auto 1 per-group
run 4096x11008 auto 1 per-group
run 4096x11008 auto 16 per-channel
run 8192x28672 '{"ntok":16,"split":4,"csplit":2}' 16 per-group
run 11008x4096 '{"ntok":32,"split":1}' 32 per-group
run 4096x11008 auto 32 per-group
cat gpurun_out/stress.txt
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_1.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_1.log
tail -2 gpurun_out/pytest_gpu_1.log
