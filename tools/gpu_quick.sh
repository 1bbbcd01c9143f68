#!/bin/bash
# Quick GPU iteration: gpu tests, bench, optional ncu --set full of kernels matching $NCU_K.
# usage (under gpurun): NCU_K=regex bash tools/gpu_quick.sh tag
set -u
TAG=${1:-q}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py --no-cpu-baseline > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
python tools/bench_summary.py $OUT/bench_$TAG.json
if [ -n "${NCU_K:-}" ]; then
python tools/prof_step.py --config 4 --warmup 2 --steps 1 > $OUT/plain_$TAG.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:${NCU_K}" -s ${NCU_S:-0} -c ${NCU_C:-4} \
    -o $OUT/prof_$TAG python tools/prof_step.py --config 4 --warmup 2 --steps 1 \
    > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
