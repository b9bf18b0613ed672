#!/bin/bash
# bench lines for BASELINE configs 2, 4, 5 and the mode comparison (naive / fifo / infinite / full)
OUT=gpurun_out/${1:-cfg}
mkdir -p $OUT
for c in 2 4 5; do
  timeout 900 python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline > $OUT/bench_c$c.json 2> $OUT/bench_c$c.err
done
timeout 900 python tools/modes_compare.py --config 3 --prompts 2 > $OUT/modes_c3.json 2> $OUT/modes_c3.err
timeout 900 python tools/modes_compare.py --config 2 --prompts 4 > $OUT/modes_c2.json 2> $OUT/modes_c2.err
timeout 900 python tools/modes_compare.py --config 4 --prompts 2 > $OUT/modes_c4.json 2> $OUT/modes_c4.err
echo done > $OUT/DONE
