set -u
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
for rep in 1 2 3; do python tools/stage_bench_cfg.py 4 40 2>/dev/null; done
python tools/stage_bench_cfg.py 5 10 2>/dev/null
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -k "rhs or fluid or config_step" > gpurun_out/pytest_r2h.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_r2h.log
