#!/bin/bash
OUT=gpurun_out/${1:-sweep}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
for cfg in "WARM=20" "WARM=600" "WARM=300 GROUPS=8" "WARM=300 GROUPS=4"; do
  echo "$cfg" >> $OUT/sweep.txt; env $cfg IMPL=1 timeout 300 python tools/mk_step_time.py >> $OUT/sweep.txt 2>&1
done
