#!/bin/bash
OUT=gpurun_out/${1:-det}
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest.log 2>&1; echo "rc=$?" >> $OUT/pytest.log
timeout 1200 python tools/modes_compare.py --config 3 --prompts 2 > $OUT/modes_c3.json 2>&1
timeout 1200 python tools/modes_compare.py --config 4 --prompts 2 > $OUT/modes_c4.json 2>&1
echo done > $OUT/DONE
