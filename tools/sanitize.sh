#!/bin/bash
# compute-sanitizer over the tiny config (smoke: prefill + FPTAS/SJF continuous-sampling rollout,
# eager steps so every launch is checked) and the split-attention hook: memcheck, racecheck,
# synccheck.  Logs under gpurun_out/<tag>/.
TAG=${1:-sanitize}
OUT=gpurun_out/$TAG
mkdir -p $OUT
for tool in memcheck racecheck synccheck; do
  IS_NO_GRAPH=1 timeout 1200 compute-sanitizer --tool $tool --print-limit 50 \
    python -c "import __graft_entry__ as g; g.smoke()" > $OUT/$tool.smoke.log 2>&1
  echo "rc=$?" >> $OUT/$tool.smoke.log
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 \
    python tools/attn_bench.py --impls 0 --reps 1 --case config3_g8 > $OUT/$tool.attn.log 2>&1
  echo "rc=$?" >> $OUT/$tool.attn.log
done
echo done > $OUT/DONE
