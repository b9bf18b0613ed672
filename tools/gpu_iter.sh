#!/bin/bash
# Short iteration call: GPU tests (optionally filtered), one bench line, smoke.
TAG=${1:-iter}
FILTER=${2:-}
OUT=gpurun_out/$TAG
mkdir -p $OUT
if [ -n "$FILTER" ]; then
  timeout 900 python -m pytest tests -m gpu -x -q -k "$FILTER" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
else
  timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
fi
timeout 600 python bench.py --no-cpu-baseline > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?" >> $OUT/bench.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
echo done > $OUT/DONE
