timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_stress.py -q -x -p no:cacheprovider -k "cluster_splitk_128 or repeated" > gpurun_out/pytest_q.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_q.log
tail -3 gpurun_out/pytest_q.log
LIBS="prod csbdsmem" QB="--shapes 4096x4096,11008x4096 --ms 32,64,128,256 --cfgs auto;{\"ntok\":128,\"split\":4,\"csplit\":2};{\"ntok\":128,\"split\":4,\"csplit\":4}" bash scripts/gpu_abq.sh
