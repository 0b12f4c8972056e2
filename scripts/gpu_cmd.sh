timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu_1.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu_1.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
SAN_TIMEOUT=900 bash scripts/sanitize.sh > /dev/null 2>&1
true
