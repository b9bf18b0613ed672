#!/bin/bash
OUT=gpurun_out/${1:-grp}
mkdir -p $OUT
for m in 2 4 8; do
  timeout 900 python bench.py --groups $m --steps 1 --warmup 3 > $OUT/bench_g$m.json 2> $OUT/bench_g$m.err
done
echo done > $OUT/DONE
