timeout 900 python -m pytest tests/test_pipeline.py tests/test_gpu_parity.py -q -p no:cacheprovider -k "smooth or pipeline or quant or apply" > gpurun_out/pytest_q.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q.log
tail -3 gpurun_out/pytest_q.log; grep -m5 "Error\|assert" gpurun_out/pytest_q.log
timeout 600 python scripts/c4_probe.py > gpurun_out/c4_probe.txt 2>&1; cat gpurun_out/c4_probe.txt
