#!/bin/bash
OUT=gpurun_out/${1:-ncuattn}
mkdir -p $OUT
# 8 co-resident groups after ~290 steps: full captures of one layer's prefix + suffix kernels
env GROUPS=8 IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:attn_(prefix|suffix)' -s 16300 -c 2 -o $OUT/attn_g8 python tools/step_driver.py --steps 300 > $OUT/ncu_g8.log 2>&1
echo done > $OUT/DONE
