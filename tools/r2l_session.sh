set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke_r2l.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/smoke_r2l.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q -k "spread or interp or config_step or small_sheet or window or force or degenerate or slab" > gpurun_out/pytest_r2l.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_r2l.log
bash tools/build_variants.sh fma "-DIBK_SPMMA=0" mma5 "-DIBK_SP_MINB=5" mma6 "-DIBK_SP_MINB=6" mma4 "-DIBK_SP_MINB=4" > gpurun_out/variants_r2l.log 2>&1
for rep in 1 2; do
for v in fma default mma4 mma5 mma6; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4 30 2>/dev/null | sed "s/^/$v /"
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4h 30 2>/dev/null | sed "s/^/$v /"
done
done
