#!/bin/bash
# ncu --set full (with source) of the decode GEMMs at config 3, step 2: QKV (EPI 4), o_proj and down
# (EPI 1: launches alternate o, down per layer), gate/up (EPI 2), lm_head (EPI 3).
OUT=gpurun_out/${1:-ncugemm}
mkdir -p $OUT
for spec in "4:qkv:28" "1:oproj_down:56" "3:lmhead:1"; do
  e=${spec%%:*}; rest=${spec#*:}; name=${rest%%:*}; skip=${rest#*:}
  IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
    -k "regex:gemm_swapab_kernel<\(int\)16, \(int\)$e" -s $skip -c 2 -o $OUT/$name python tools/step_driver.py --steps 2 \
    > $OUT/ncu_$name.log 2>&1
done
python tools/summarize_profiles.py $OUT $OUT/summary 0 > $OUT/summary.log 2>&1
for r in $OUT/*.ncu-rep; do python tools/ncu_stalls.py $r "" 15 > ${r%.ncu-rep}.stalls.txt 2>&1; done
mkdir -p /tmp/ncu_reps && mv $OUT/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
echo done > $OUT/DONE
