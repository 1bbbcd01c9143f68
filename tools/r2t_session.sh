python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 600 python -m pytest tests -m "gpu and not slow" -x -q -k "rhs or fluid or config_step or anisotropic or z512" > gpurun_out/pytest_r2t.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_r2t.log
bash tools/build_variants.sh pf0 "-DIBK_XZPF=0" pf2 "-DIBK_XZPF=2" pf8 "-DIBK_XZPF=8" > /dev/null 2>&1
for rep in 1 2; do
for v in pf0 pf2 default pf8; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4 30 2>/dev/null | sed "s/^/$v /"
done
done
for v in pf0 pf2 default pf8; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4h 30 2>/dev/null | sed "s/^/$v /"
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 5 8 2>/dev/null | sed "s/^/$v /"
done
