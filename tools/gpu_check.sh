#!/bin/bash
# GPU check: smoke, full pytest -m gpu (with durations), one bench line.
# usage (under gpurun): bash tools/gpu_check.sh tag [pytest -k expr]
set -u
TAG=${1:-chk}
K=${2:-}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
if [ -n "$K" ]; then
  timeout 2400 python -m pytest tests -m gpu -x -q -s --durations=25 -k "$K" > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
else
  timeout 2400 python -m pytest tests -m gpu -x -q -s --durations=25 > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
fi
tail -40 $OUT/pytest_gpu_$TAG.log | grep -v "^$" | tail -32
if [ "${NO_BENCH:-0}" != "1" ]; then
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
python tools/bench_summary.py $OUT/bench_$TAG.json
fi
