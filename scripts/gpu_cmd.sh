timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "pair_tiles" > gpurun_out/pytest_q.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q.log
tail -3 gpurun_out/pytest_q.log; grep -m3 "Error" gpurun_out/pytest_q.log
timeout 600 python scripts/quick_bench.py --shapes 4096x11008,4096x4096,11008x4096 --ms 256,512,1024 --fp16 --cfgs 'auto;{"ntok":256,"split":3};{"ntok":192,"split":3};{"ntok":192,"split":5}' > gpurun_out/qb.txt 2>&1
true
