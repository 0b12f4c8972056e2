# quick GPU iteration: parity subset + chain timelines + decode points
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -p no:cacheprovider ${PYTEST_ARGS} > gpurun_out/pytest_quick.log 2>&1
echo "pytest exit $?" >> gpurun_out/pytest_quick.log
tail -3 gpurun_out/pytest_quick.log
for spec in ${SPECS:-4096x4096/1}; do
  IFS=/ read shape m <<< "$spec"
  QQQ_LIB_PATH=paper_2406_09904_b200/lib/libqqq_b200_tl.so timeout 120 python scripts/chain_timeline.py --shape $shape --m $m --len 6 ${TLARGS} >> gpurun_out/chain_tl.txt 2>&1
done
[ -n "$QB" ] && timeout 600 python scripts/quick_bench.py $QB > gpurun_out/quick_bench.txt 2>&1
true
