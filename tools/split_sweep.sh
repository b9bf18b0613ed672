#!/bin/bash
OUT=gpurun_out/${1:-split}
mkdir -p $OUT
run() { echo "$1" >> $OUT/sweep.txt; env $1 IMPL=1 timeout 300 python tools/mk_step_time.py 2>&1 | head -1 >> $OUT/sweep.txt; }
run "IS_X=0"
run "IS_STG_QKV=6"
run "IS_STG_QKV=8"
run "IS_STG_O=6"
run "IS_STG_GU=6"
run "IS_STG_D=6"
run "IS_STG_D=8"
run "IS_STG_QKV=6 IS_STG_D=6"
run "IS_X=0"
