python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
python tools/l2_probe.py
timeout 600 python -m pytest tests/test_slab.py -m gpu -q -k window > gpurun_out/pytest_r2n.log 2>&1; echo "slab window rc=$?"; tail -1 gpurun_out/pytest_r2n.log
