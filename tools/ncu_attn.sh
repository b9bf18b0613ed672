#!/bin/bash
OUT=gpurun_out/${1:-ncuattn}
mkdir -p $OUT
# 8 groups, after 300 steps: full captures of one layer's prefix + suffix kernels
env GROUPS=8 IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:attn' -s 16900 -c 2 -o $OUT/attn_g8 python tools/step_driver.py --steps 302 > $OUT/ncu_g8.log 2>&1
GROUPS=1 IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:attn' -s 33700 -c 2 -o $OUT/attn_g1 python tools/step_driver.py --steps 602 > $OUT/ncu_g1.log 2>&1
echo done > $OUT/DONE
