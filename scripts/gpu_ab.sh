# A/B chain timelines: LIBS="name1 name2" (lib/<name>.so; 'tl' = libqqq_b200_tl.so), SPECS, TLARGS
mkdir -p gpurun_out
for name in ${LIBS:-tl}; do
  lib=paper_2406_09904_b200/lib/$name.so; [ "$name" = tl ] && lib=paper_2406_09904_b200/lib/libqqq_b200_tl.so
  for spec in ${SPECS:-4096x4096/1}; do
    IFS=/ read shape m <<< "$spec"
    echo "=== lib $name" >> gpurun_out/chain_tl.txt
    QQQ_LIB_PATH=$lib timeout 120 python scripts/chain_timeline.py --shape $shape --m $m --len 6 ${TLARGS} >> gpurun_out/chain_tl.txt 2>&1
  done
done
true
