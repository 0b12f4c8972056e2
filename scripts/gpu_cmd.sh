QQQ_LIB_PATH=paper_2406_09904_b200/lib/nbar.so timeout 600 compute-sanitizer --tool racecheck --racecheck-report all --print-limit 10 python scripts/sanitize_cases.py --quick > gpurun_out/racecheck_nbar.txt 2>&1; echo "exit $?" >> gpurun_out/racecheck_nbar.txt
grep -v "^=========     \|Host Frame\|^========= $" gpurun_out/racecheck_nbar.txt | tail -14
LIBS="prod nbar" QB="--shapes 4096x4096,4096x11008 --ms 1,16,128,1024" bash scripts/gpu_abq.sh
