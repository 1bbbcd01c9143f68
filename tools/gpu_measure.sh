#!/bin/bash
# Measurement session: bench lines for every config, ncu launch list + --set full of one
# step per config (for profiles/ncu_traffic_cfg<k>.json), experiments JSON.
# usage (under gpurun): bash tools/gpu_measure.sh tag "1 2 3 4 5 4h"
set -u
TAG=${1:-m}
CFGS=${2:-"1 2 3 4 5 4h"}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build rc=$?"
for c in $CFGS; do
  if [ "$c" = "4" ]; then CPUB=""; else CPUB="--no-cpu-baseline"; fi
  timeout 900 python bench.py --config $c $CPUB > $OUT/bench_${TAG}_cfg$c.json 2> $OUT/bench_${TAG}_cfg$c.err; echo "bench cfg$c rc=$?"
done
# per-step launches: create (3 table launches) + bin (5) + per step 8 (+1 drive)
for c in $CFGS; do
  python tools/prof_step.py --config $c --warmup 2 --steps 1 > $OUT/plain_${TAG}_cfg$c.log 2>&1 || continue
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_${TAG}_cfg$c.csv python tools/prof_step.py --config $c --warmup 2 --steps 1 \
      > $OUT/ncu_launch_${TAG}_cfg$c.log 2>&1; echo "ncu launches cfg$c rc=$?"
  # --set full of the last step's kernels (skip create + bin + 2 warm-up steps)
  NL=$(grep -c gpu__time_duration $OUT/launches_${TAG}_cfg$c.csv)
  PER=8
  SKIP=$(( NL - PER ))
  timeout 1500 ncu --set full --clock-control none --import-source on -s $SKIP -c $PER \
      -o $OUT/prof_${TAG}_cfg$c python tools/prof_step.py --config $c --warmup 2 --steps 1 \
      > $OUT/ncu_full_${TAG}_cfg$c.log 2>&1; echo "ncu full cfg$c rc=$?"
  # summaries on the box (gpurun copies back at most 64 MiB): profiles_out/, then drop the
  # report unless it is cfg4's
  mkdir -p $OUT/profiles_out
  PROF_OUT=$OUT/profiles_out python tools/make_profiles.py ${TAG}_cfg$c $c > /dev/null 2>&1
  if [ "$c" != "4" ]; then rm -f $OUT/prof_${TAG}_cfg$c.ncu-rep; fi
done
if [ "${EXPER:-1}" = "1" ]; then
  timeout 900 python -m paper_math_0301321_b200.experiments sweep --steps 1600 --periods 50,100,200,400 > $OUT/sweep_$TAG.json 2> $OUT/sweep_$TAG.err; echo "sweep rc=$?"
  timeout 600 python -m paper_math_0301321_b200.experiments linearity --steps 400 > $OUT/linearity_$TAG.json 2> $OUT/linearity_$TAG.err; echo "linearity rc=$?"
  timeout 900 python -m pytest tests -m gpu -x -q -s -k "strip_experiment or time_coupling" > $OUT/pytest_exp_$TAG.log 2>&1; echo "pytest exp rc=$?"; tail -3 $OUT/pytest_exp_$TAG.log
fi
ls $OUT/profiles_out
du -sh $OUT
if [ $(du -sm $OUT | cut -f1) -gt 60 ]; then rm -f $OUT/*.ncu-rep; fi
