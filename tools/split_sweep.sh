#!/bin/bash
OUT=gpurun_out/${1:-split}
mkdir -p $OUT
for k in 1 4 8 1; do
  echo "K=$k" >> $OUT/sweep.txt
  IS_STEPS_PER_GRAPH=$k timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['ms_per_decode_step'], d['decode_steps_per_rollout'])" >> $OUT/sweep.txt 2>&1
done
