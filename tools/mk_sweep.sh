#!/bin/bash
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
echo "per-op" >> $OUT/sweep.txt; IMPL=1 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
echo "per-op separate merge" >> $OUT/sweep.txt; IS_SEPARATE_MERGE=1 IMPL=1 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
echo "persistent" >> $OUT/sweep.txt; IMPL=0 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
IS_TIMELINE=1 timeout 300 python tools/step_driver.py --steps 30 > $OUT/timeline.txt 2>&1
