#!/bin/bash
OUT=gpurun_out/${1:-split}
mkdir -p $OUT
IS_BNORM=qkv timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q -k "per_op or fullsize" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
run() { echo "$1" >> $OUT/sweep.txt; env $1 IMPL=1 timeout 300 python tools/mk_step_time.py 2>&1 | head -1 >> $OUT/sweep.txt; }
run "IS_X=0"
run "IS_BNORM=qkv"
run "IS_BNORM=1"
run "IS_X=0"
run "IS_BNORM=qkv"
