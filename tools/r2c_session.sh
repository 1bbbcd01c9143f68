set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_r2c.log 2>&1; echo "build rc=$?"
timeout 1200 python -m pytest tests/test_slab.py -m gpu -x -q -s > gpurun_out/pytest_slab_r2c.log 2>&1; echo "slab rc=$?"; tail -3 gpurun_out/pytest_slab_r2c.log
bash tools/build_variants.sh base "-DIBK_ZHOIST=0 -DIBK_XSWAP=0" zh "-DIBK_XSWAP=0" xs "-DIBK_ZHOIST=0" > gpurun_out/variants_r2c.log 2>&1
for rep in 1 2; do
for v in base zh xs default; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4 40 2>/dev/null | sed "s/^/$v /"
done
done
for v in base default; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 5 10 2>/dev/null | sed "s/^/$v /"
done
