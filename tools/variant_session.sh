#!/bin/bash
# Dev A/B session (under gpurun): build -D variants of the library, run a parity subset on
# the default build, then alternate per-stage timings of every variant.
# usage: VARIANTS="x0:-DIBK_XSEL=0 x1:-DIBK_XSEL=1" CFGS="4 5" REPS=2 K="fluid or rhs" \
#        bash tools/variant_session.sh tag
set -u
TAG=${1:-v}
OUT=gpurun_out
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build_$TAG.log 2>&1; echo "build rc=$?"
if [ -n "${K:-}" ]; then
  timeout 1200 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest_$TAG.log 2>&1; echo "pytest rc=$?"
  tail -1 $OUT/pytest_$TAG.log
fi
NAMES=""
for v in ${VARIANTS:-}; do
  n=${v%%:*}; f=${v#*:}
  # "name" alone: a prebuilt build_variants/name.so shipped with the snapshot
  if [ "$n" != "$v" ]; then bash tools/build_variants.sh $n "${f//,/ }" > /dev/null 2>&1; fi
  NAMES="$NAMES $n"
done
for rep in $(seq 1 ${REPS:-2}); do
  for c in ${CFGS:-4}; do
    for v in $NAMES default; do
      if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
      IB_B200_LIB=$L timeout 300 python tools/stage_bench_cfg.py $c ${STEPS:-20} 2>/dev/null | \
        python -c "import sys,json; d=json.loads(sys.stdin.read()); print('$v', 'cfg$c', d['graph_ms'], d['stages_us'])"
    done
  done
done
if [ -n "${NCU_K:-}" ]; then
  python tools/prof_step.py --config ${NCU_CFG:-4} --warmup 2 --steps 1 > /dev/null 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:${NCU_K}" -s ${NCU_S:-0} -c ${NCU_C:-1} \
      -o $OUT/prof_$TAG python tools/prof_step.py --config ${NCU_CFG:-4} --warmup 2 --steps 1 \
      > $OUT/ncu_full_$TAG.log 2>&1; echo "ncu full rc=$?"
fi
