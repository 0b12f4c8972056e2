#!/bin/bash
# one development iteration on the GPU box: parity tests, quick sweep, timeline
mkdir -p gpurun_out
rm -f gpurun_out/iter_*.log
timeout 600 python -m pytest tests -m gpu -x -q --timeout 300 -p no:cacheprovider > gpurun_out/iter_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/iter_pytest.log
timeout 600 python scripts/quick_bench.py --shapes ${SHAPES:-4096x4096,4096x11008,11008x4096} --ms ${MS:-1,16,64,128,256,512,1024} ${QARGS} > gpurun_out/iter_quick.log 2>&1
echo "quick exit $?" >> gpurun_out/iter_quick.log
for spec in ${TL}; do
  echo "== $spec" >> gpurun_out/iter_timeline.log
  timeout 120 python scripts/timeline.py $(echo $spec | tr ':' ' ') >> gpurun_out/iter_timeline.log 2>&1
done
tail -3 gpurun_out/iter_pytest.log; cat gpurun_out/iter_quick.log
