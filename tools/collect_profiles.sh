#!/bin/bash
# After `gpurun -- bash tools/measure_session.sh TAG` has merged gpurun_out/: copy the
# session's summaries into profiles/ (tracked).  usage: bash tools/collect_profiles.sh TAG
set -eu
T=${1:?tag}
O=gpurun_out
cp $O/profiles_out/* profiles/
grep -o "\[{'cfg'.*\]" $O/pytest_gpu_$T.log > profiles/${T}_parity_reports.txt
tail -3 $O/pytest_gpu_$T.log > profiles/${T}_gpu_suite.txt
cp $O/bench_ref_$T.json profiles/${T}_reference_arm.json
cp $O/bench_slab_$T.json profiles/${T}_slab4_bench.json
cp $O/bench_slabf_$T.json profiles/${T}_slab4_fused_bench.json
[ -s $O/sweep_$T.json ] && cp $O/sweep_$T.json profiles/${T}_sweep_cfg3.json
[ -s $O/linearity_$T.json ] && cp $O/linearity_$T.json profiles/${T}_linearity_cfg3.json
[ -f $O/prof_${T}_cfg4.ncu-rep ] && python tools/ncu_pipes.py $O/prof_${T}_cfg4.ncu-rep > profiles/${T}_cfg4_pipes.txt 2>&1
for c in 1 2 3 4 4h 5; do python tools/bench_summary.py $O/bench_${T}_cfg$c.json 2>/dev/null | sed -n 1p | sed "s/^/cfg$c /"; done
wc -l profiles/${T}_parity_reports.txt
