set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2d.log 2>&1; echo "build rc=$?"
timeout 300 python tools/slab_debug.py 4 2>&1 | tail -40
timeout 300 python tools/slab_debug.py 2 2>&1 | tail -20
