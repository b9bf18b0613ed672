#!/bin/bash
# K5 microbenchmark + ncu captures of both decode attention kernels (>= 32 MB launches).
TAG=${1:-attn}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 python tools/attn_bench.py --impls 0,1,2 > $OUT/attn_bench.jsonl 2> $OUT/attn_bench.err
# full ncu captures of the attention launches: 8 groups x 8 rows x 1024 tokens (157 MB), and config 3
for c in groups8_t1024 config3_g8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:attn_(prefix|suffix|kernel|merge)' -c 6 \
    -o $OUT/k5_$c python tools/attn_bench.py --impls 0 --reps 1 --case $c > $OUT/ncu_$c.log 2>&1
done
python tools/summarize_profiles.py $OUT $OUT/summary 60 > $OUT/summary.log 2>&1
echo done > $OUT/DONE
