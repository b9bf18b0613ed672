#!/bin/bash
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
echo "nodeps pf2" >> $OUT/sweep.txt; IS_MK_NODEPS=1 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
echo "nodeps pf0" >> $OUT/sweep.txt; IS_MK_NODEPS=1 IS_MK_PF=0 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
echo "per-op" >> $OUT/sweep.txt; IMPL=1 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
