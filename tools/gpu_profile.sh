#!/bin/bash
# Profile capture for profiles/: bench line, ncu launch list and ncu --set full of one cfg4
# step (after 2 warm-up steps).  Launch order: 1 (tables) + 5 (cell binning) + 9 per step.
# usage (under gpurun): bash tools/gpu_profile.sh tag
set -u
TAG=${1:-prof}
OUT=gpurun_out
mkdir -p $OUT
python bench.py > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
python tools/prof_step.py --config 4 --warmup 2 --steps 1 > $OUT/plain_$TAG.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -s 24 -c 9 --csv \
    --log-file $OUT/launches_$TAG.csv python tools/prof_step.py --config 4 --warmup 2 --steps 1 \
    > $OUT/ncu_launch_$TAG.log 2>&1; echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -s 24 -c 9 \
    -o $OUT/prof_$TAG python tools/prof_step.py --config 4 --warmup 2 --steps 1 \
    > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
