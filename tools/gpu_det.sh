#!/bin/bash
OUT=gpurun_out/${1:-det}
mkdir -p $OUT
timeout 600 python tools/modes_compare.py --config 3 --prompts 1 --modes infinite,infinite > $OUT/inf_inf.json 2>&1
timeout 600 python tools/modes_compare.py --config 3 --prompts 1 --modes naive,infinite > $OUT/naive_inf.json 2>&1
IS_SEPARATE_MERGE=1 timeout 600 python tools/modes_compare.py --config 3 --prompts 1 --modes naive,infinite > $OUT/naive_inf_sepmerge.json 2>&1
IS_NO_TC_PREFIX=1 timeout 600 python tools/modes_compare.py --config 3 --prompts 1 --modes naive,infinite > $OUT/naive_inf_notc.json 2>&1
echo done > $OUT/DONE
