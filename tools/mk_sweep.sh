#!/bin/bash
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
for w in 20 300 600 900; do
  echo "warm=$w" >> $OUT/sweep.txt; WARM=$w IMPL=1 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
done
