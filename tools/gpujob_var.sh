# time variant libraries (tools/variants.py) on the given configs: fwd_topk / step per variant
for v in ${VARIANTS}; do
  lib=varlib/$v.so; [ "$v" = product ] && lib=paper_2501_14577_b200/libonedf.so
  for c in ${CONFIGS:-long64k}; do
    echo "$v $c $(ONEDF_LIB=$PWD/$lib timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu --no-e2e 2>/dev/null | tail -1)" >> gpurun_out/variants.txt
  done
done
