#!/bin/bash
# Full measurement session (under gpurun): smoke, the whole GPU suite, then for every config
# a bench line, an ncu launch list and an ncu --set full summary (tools/gpu_measure.sh),
# the reference arm and the slab line.
# usage: bash tools/measure_session.sh tag
set -u
TAG=${1:-m}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_$TAG.log
timeout 2400 python -m pytest tests -m gpu -q -s --durations=15 > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu_$TAG.log | tail -2
EXPER=${EXPER:-1} bash tools/gpu_measure.sh $TAG "4 1 2 3 5 4h"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; echo "ref rc=$?"
timeout 600 python bench.py --mode slab --slab-P 4 --steps 20 --warmup 3 > gpurun_out/bench_slab_$TAG.json 2> gpurun_out/bench_slab_$TAG.err; echo "slab rc=$?"
timeout 600 python bench.py --mode slab --slab-P 4 --slab-fused --steps 20 --warmup 3 > gpurun_out/bench_slabf_$TAG.json 2> gpurun_out/bench_slabf_$TAG.err; echo "slab fused rc=$?"
# launch list of the bench command itself (cold-cache, serialised: compare shares, not times)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/launches_${TAG}b.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline \
    > gpurun_out/ncu_launch_${TAG}b.log 2>&1; echo "ncu bench launches rc=$?"
mkdir -p gpurun_out/profiles_out
PROF_OUT=gpurun_out/profiles_out python tools/make_profiles.py ${TAG}b 4 > /dev/null 2>&1; echo "summary rc=$?"
