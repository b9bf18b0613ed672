#!/bin/bash
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "per_op or gemm" > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
echo "per-op" >> $OUT/sweep.txt; IMPL=1 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
IS_TIMELINE=1 timeout 300 python tools/step_driver.py --steps 30 > $OUT/timeline.txt 2>&1
