# A/B of quick_bench across library variants: LIBS="prod name ..." (lib/<name>.so), QB="quick_bench args"
mkdir -p gpurun_out
for name in ${LIBS:-prod}; do
  lib=paper_2406_09904_b200/lib/$name.so; [ "$name" = prod ] && lib=paper_2406_09904_b200/lib/libqqq_b200.so
  echo "=== lib $name" >> gpurun_out/abq.txt
  QQQ_LIB_PATH=$lib timeout 600 python scripts/quick_bench.py $QB >> gpurun_out/abq.txt 2>&1
done
true
