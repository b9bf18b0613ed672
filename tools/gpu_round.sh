#!/bin/bash
# One gpurun call: GPU tests, bench line, smoke, launch list and full ncu captures of the top kernels.
# usage (from this container):  gpurun --timeout 2400 -- 'bash tools/gpu_round.sh [tag]'
TAG=${1:-r01}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/gpu.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
# launch list of eager decode steps after prefill (cold-cache, serialised: compare shares)
IS_NO_GRAPH=1 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file $OUT/launches.csv python tools/step_driver.py --steps 3 > $OUT/launches.log 2>&1
# full captures: gate/up GEMM (EPI_SWIGLU = 2), the suffix attention kernel, the tcgen05 prefix kernel
IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_swapab_kernel<\(int\)16, \(int\)2' -s 28 -c 2 -o $OUT/gateup python tools/step_driver.py --steps 2 > $OUT/ncu_gateup.log 2>&1
IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on \
  -k 'regex:attn' -s 56 -c 4 -o $OUT/attn python tools/step_driver.py --steps 2 > $OUT/ncu_attn.log 2>&1
IS_NO_GRAPH=1 timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k 'regex:gemm_swapab_kernel<\(int\)16, \(int\)3' -s 0 -c 1 -o $OUT/lmhead python tools/step_driver.py --steps 2 > $OUT/ncu_lmhead.log 2>&1
# counters of the captures summarised here (ncu is on this box), the large .ncu-rep files kept
# out of gpurun_out/ (the merge back is capped at 64 MiB)
python tools/summarize_profiles.py $OUT $OUT/summary 60 > $OUT/summary.log 2>&1
mkdir -p /tmp/ncu_reps && mv $OUT/*.ncu-rep /tmp/ncu_reps/ 2>/dev/null
for f in $OUT/*.log $OUT/*.csv; do [ -f "$f" ] && [ $(stat -c %s "$f") -gt 8000000 ] && gzip -f "$f"; done
echo done > $OUT/DONE
