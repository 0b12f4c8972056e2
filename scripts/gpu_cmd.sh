SAN_TIMEOUT=700 bash scripts/sanitize.sh > gpurun_out/san_summary.txt 2>&1
cat gpurun_out/san_summary.txt
