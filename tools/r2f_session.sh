set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build_r2f.log 2>&1; echo "build+smoke rc=$?"; tail -2 gpurun_out/build_r2f.log
timeout 1500 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_r2f.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_r2f.log
for c in 4 4h 5; do python tools/stage_bench_cfg.py $c 30 2>/dev/null; done
