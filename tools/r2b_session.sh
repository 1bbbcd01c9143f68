set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2b.log 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_slab.py -m gpu -x -q -s > gpurun_out/pytest_slab_r2b.log 2>&1; echo "slab rc=$?"; tail -5 gpurun_out/pytest_slab_r2b.log
NO_BENCH=1 bash tools/gpu_check.sh r2b
EXPER=1 bash tools/gpu_measure.sh r2m "1 2 3 4 5 4h"
