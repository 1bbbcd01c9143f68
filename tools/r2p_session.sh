python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "z512 or fft or fluid or project or rings" > gpurun_out/pytest_r2p.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_r2p.log
bash tools/build_variants.sh c4 "-DIBK_Z512C=4" > /dev/null 2>&1
for v in c4 default c4 default; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 5 10 2>/dev/null | sed "s/^/$v /"
done
