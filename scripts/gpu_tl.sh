# chain timelines for the decode A/B variants: VARIANTS="name:cfgjson ..." SPECS="shape/m ..."
mkdir -p gpurun_out
for v in ${VARIANTS:-tl:{}}; do
  name=${v%%:*}; cfg=${v#*:}
  lib=paper_2406_09904_b200/lib/$name.so; [ "$name" = tl ] && lib=paper_2406_09904_b200/lib/libqqq_b200_tl.so
  for spec in ${SPECS:-4096x4096/1}; do
    IFS=/ read shape m <<< "$spec"
    echo "=== variant $name cfg $cfg" >> gpurun_out/chain_tl.txt
    QQQ_LIB_PATH=$lib timeout 120 python scripts/chain_timeline.py --shape $shape --m $m --len 6 --cfg "$cfg" >> gpurun_out/chain_tl.txt 2>&1
  done
done
cat gpurun_out/chain_tl.txt
