python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r2r.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2r.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_r2r.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_r2r.log
for c in 4 4 5 4h 3; do python tools/stage_bench_cfg.py $c 30 2>/dev/null; done
