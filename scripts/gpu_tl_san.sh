mkdir -p gpurun_out
for spec in 4096x4096/1 4096x11008/1 4096x11008/16 11008x4096/1; do
  IFS=/ read shape m <<< "$spec"
  timeout 120 python scripts/chain_timeline.py --shape $shape --m $m --len 6 >> gpurun_out/chain_tl.txt 2>&1
done
timeout 120 python scripts/chain_timeline.py --shape 4096x4096 --m 1 --len 6 --scheme per-channel >> gpurun_out/chain_tl.txt 2>&1
SAN_TIMEOUT=600 bash scripts/sanitize.sh
cat gpurun_out/chain_tl.txt
