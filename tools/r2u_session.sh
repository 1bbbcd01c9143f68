python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r2u.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2u.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_r2u.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_r2u.log
bash tools/build_variants.sh yr0 "-DIBK_YREGTW=0" > /dev/null 2>&1
for rep in 1 2; do
for v in yr0 default; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4 30 2>/dev/null | sed "s/^/$v /"
done
done
for v in yr0 default; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4h 30 2>/dev/null | sed "s/^/$v /"
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 3 30 2>/dev/null | sed "s/^/$v /"
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 5 8 2>/dev/null | sed "s/^/$v /"
done
