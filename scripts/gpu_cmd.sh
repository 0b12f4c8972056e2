QQQ_LIB_PATH=paper_2406_09904_b200/lib/lsu.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "gemm" > gpurun_out/pytest_q.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q.log
tail -2 gpurun_out/pytest_q.log; grep -m3 "Error" gpurun_out/pytest_q.log
LIBS="prod lsu prod lsu" QB="--shapes 4096x4096,4096x11008,11008x4096 --ms 1,16,32" bash scripts/gpu_abq.sh
