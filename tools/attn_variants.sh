#!/bin/bash
# K5 microbenchmark under attention launch variants (carveout / suffix shape), one line per case.
OUT=${1:-gpurun_out/attnvar}
mkdir -p $OUT
for v in "" "IS_ATTN_CARVEOUT=100" "IS_SUFFIX_SHAPE=1" "IS_ATTN_CARVEOUT=100 IS_SUFFIX_SHAPE=1"; do
  echo "# $v" >> $OUT/attn_variants.jsonl
  env $v timeout 300 python tools/attn_bench.py --impls 0 --reps 10 >> $OUT/attn_variants.jsonl 2>&1
done
