set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2e.log 2>&1; echo "build rc=$?"
timeout 1500 python -m pytest tests/test_slab.py -m gpu -q -s > gpurun_out/pytest_slab_r2e.log 2>&1; echo "slab rc=$?"; tail -3 gpurun_out/pytest_slab_r2e.log
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "spread or interp or force or config_step or window or small_sheet" > gpurun_out/pytest_lag_r2e.log 2>&1; echo "lag rc=$?"; tail -2 gpurun_out/pytest_lag_r2e.log
bash tools/build_variants.sh sp1 "-DIBK_SPMAP=1" x512 "-DIBK_XRB512=64" > gpurun_out/variants_r2e.log 2>&1
for rep in 1 2; do
for v in sp1 default; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4 40 2>/dev/null | sed "s/^/$v /"
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4h 40 2>/dev/null | sed "s/^/$v /"
done
done
for v in x512 default; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 5 10 2>/dev/null | sed "s/^/$v /"
done
timeout 300 python bench.py --mode slab --slab-P 4 --steps 20 --warmup 3 > gpurun_out/bench_slab_r2e.json 2>gpurun_out/bench_slab_r2e.err; echo "slab bench rc=$?"; cat gpurun_out/bench_slab_r2e.json
