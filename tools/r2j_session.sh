set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r2j.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2j.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_r2j.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_r2j.log
bash tools/build_variants.sh cz1 "-DIBK_XCZ=1" cz4 "-DIBK_XCZ=4" cz8 "-DIBK_XCZ=8" > gpurun_out/variants_r2j.log 2>&1
for rep in 1 2; do
for v in cz1 default cz4 cz8; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4 40 2>/dev/null | sed "s/^/$v /"
done
done
for v in cz1 default cz4; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 5 10 2>/dev/null | sed "s/^/$v /"
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4h 40 2>/dev/null | sed "s/^/$v /"
done
