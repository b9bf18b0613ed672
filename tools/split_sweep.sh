#!/bin/bash
OUT=gpurun_out/${1:-split}
mkdir -p $OUT
run() { echo "$1" >> $OUT/sweep.txt; env $1 IMPL=1 timeout 300 python tools/mk_step_time.py 2>&1 | head -1 >> $OUT/sweep.txt; }
run "IS_X=0"
run "IS_SPLIT_GU=2"
run "IS_SPLIT_GU=3"
run "IS_SPLIT_D=4"
run "IS_SPLIT_D=6"
run "IS_SPLIT_QKV=2"
run "IS_SPLIT_QKV=8"
run "IS_SPLIT_O=4"
run "IS_X=0"
