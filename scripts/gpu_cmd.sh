rm -f gpurun_out/c4_probe.txt
for l in libqqq_b200 Q32 Q32R Q128; do echo "== $l" >> gpurun_out/c4_probe.txt; QQQ_LIB_PATH=paper_2406_09904_b200/lib/$l.so timeout 300 python scripts/c4_probe.py >> gpurun_out/c4_probe.txt 2>&1; done
