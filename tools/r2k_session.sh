set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r2k.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2k.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_r2k.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_r2k.log
for c in 4 4h 5 3; do python tools/stage_bench_cfg.py $c 30 2>/dev/null; done
for c in 4 4h; do python tools/stage_bench_cfg.py $c 30 2>/dev/null; done
