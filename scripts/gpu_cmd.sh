rm -f gpurun_out/diag.txt
python scripts/fused_diag.py 4096 4096 256 per-channel '{"ntok":128,"split":0}' >> gpurun_out/diag.txt 2>&1
python scripts/fused_diag.py 4096 4096 256 per-channel '{"ntok":256,"split":1}' >> gpurun_out/diag.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log; grep FAILED gpurun_out/pytest_gpu.log
timeout 300 python scripts/quick_bench.py --ms 1,16,128,512,1024 --shapes 4096x4096,4096x11008,11008x4096 > gpurun_out/qb.txt 2>&1
