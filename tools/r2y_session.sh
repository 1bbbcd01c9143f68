set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r2y.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2y.log
timeout 2400 python -m pytest tests -m gpu -q -s --durations=15 > gpurun_out/pytest_gpu_r2y.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" gpurun_out/pytest_gpu_r2y.log | tail -2
EXPER=0 bash tools/gpu_measure.sh r2y "4 1 2 3 5 4h"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_r2y.json 2> gpurun_out/bench_ref_r2y.err; echo "ref rc=$?"
timeout 600 python bench.py --mode slab --slab-P 4 --steps 20 --warmup 3 > gpurun_out/bench_slab_r2y.json 2> gpurun_out/bench_slab_r2y.err; echo "slab rc=$?"
