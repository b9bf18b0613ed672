#!/bin/bash
# Round-2 GPU pass: full tests, bench line (with cpu baseline), smoke, launch list, and ncu captures
# (gate/up with --cache-control all for clean traffic; attention kernels in the step at ~step 400 and
# at 8 groups; the prefix kernel's tensor pipe).
TAG=${1:-r02}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 600 python tools/attn_bench.py --impls 0,1,2 > $OUT/attn_bench.jsonl 2> $OUT/attn_bench.err
IS_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python tools/step_driver.py --steps 3 > $OUT/launches.log 2>&1
IS_NO_GRAPH=1 timeout 900 ncu --set full --cache-control all --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_swapab_kernel<\(int\)16, \(int\)2' -s 28 -c 2 -o $OUT/gateup python tools/step_driver.py --steps 2 > $OUT/ncu_gateup.log 2>&1
IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:attn_(prefix|suffix)' -s 22400 -c 4 -o $OUT/attn_step400 python tools/step_driver.py --steps 402 > $OUT/ncu_attn400.log 2>&1
env GROUPS=8 IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:attn_(prefix|suffix)' -s 16300 -c 4 -o $OUT/attn_g8 python tools/step_driver.py --steps 300 > $OUT/ncu_g8.log 2>&1
for c in groups8_t1024 config3_g8; do
  timeout 600 ncu --set full --clock-control none --import-source on -k 'regex:attn_(prefix|suffix)' -c 2 \
    -o $OUT/k5_$c python tools/attn_bench.py --impls 0 --reps 1 --case $c > $OUT/ncu_k5_$c.log 2>&1
done
python tools/summarize_profiles.py $OUT $OUT/summary 60 > $OUT/summary.log 2>&1
mkdir -p /tmp/ncu_reps && mv $OUT/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
for f in $OUT/*.log $OUT/*.csv; do [ -f "$f" ] && [ $(stat -c %s "$f") -gt 8000000 ] && gzip -f "$f"; done
echo done > $OUT/DONE
