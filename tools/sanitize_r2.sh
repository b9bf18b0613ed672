#!/bin/bash
# compute-sanitizer after the round-2 kernel changes: memcheck / synccheck over the tiny rollout
# (smoke) and over eager full-size decode steps (config 3: BN = 16, split-K GEMMs; 8 co-resident
# groups: BN = 64), racecheck of the attention hook.  Logs under gpurun_out/<tag>/.
TAG=${1:-sanitize_r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
IS_NO_GRAPH=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 50 \
  python -c "import __graft_entry__ as g; g.smoke()" > $OUT/memcheck.smoke.log 2>&1; echo "rc=$?" >> $OUT/memcheck.smoke.log
IS_NO_GRAPH=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 50 \
  python tools/step_driver.py --steps 2 > $OUT/memcheck.config3.log 2>&1; echo "rc=$?" >> $OUT/memcheck.config3.log
env GROUPS=8 IS_NO_GRAPH=1 timeout 900 compute-sanitizer --tool memcheck --print-limit 50 \
  python tools/step_driver.py --steps 2 > $OUT/memcheck.groups8.log 2>&1; echo "rc=$?" >> $OUT/memcheck.groups8.log
IS_NO_GRAPH=1 timeout 900 compute-sanitizer --tool synccheck --print-limit 50 \
  python tools/step_driver.py --steps 2 > $OUT/synccheck.config3.log 2>&1; echo "rc=$?" >> $OUT/synccheck.config3.log
timeout 900 compute-sanitizer --tool racecheck --print-limit 50 \
  python tools/attn_bench.py --impls 0 --reps 1 --case config3_g8 > $OUT/racecheck.attn.log 2>&1; echo "rc=$?" >> $OUT/racecheck.attn.log
echo done > $OUT/DONE
