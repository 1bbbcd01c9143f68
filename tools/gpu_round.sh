#!/bin/bash
# One gpurun session: GPU tests, bench, ncu launch list and ncu --set full of one cfg4 step.
# usage (under gpurun): bash tools/gpu_round.sh [tag]
set -u
TAG=${1:-r1}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu_$TAG.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?"
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"
tail -3 $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
cat $OUT/bench_$TAG.json
if [ "${NO_NCU:-0}" = "1" ]; then exit 0; fi
# launch list: ib_create = 1 launch; cfg4 step = 8 launches; skip create + 1 warm-up step
python tools/prof_step.py --config 4 --warmup 1 --steps 2 > $OUT/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 9 -c 16 --csv \
    --log-file $OUT/launches_$TAG.csv python tools/prof_step.py --config 4 --warmup 1 --steps 2 \
    > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -s 17 -c 8 \
    -o $OUT/prof_$TAG python tools/prof_step.py --config 4 --warmup 2 --steps 1 \
    > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
ls -la $OUT
