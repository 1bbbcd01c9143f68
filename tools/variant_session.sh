python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "anisotropic or fluid or rhs or fft" > gpurun_out/pytest_var.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/pytest_var.log
bash tools/build_variants.sh x0 "-DIBK_X512TMA=0" > /dev/null 2>&1
for rep in 1 2; do
for v in x0 default; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 5 8 2>/dev/null | sed "s/^/$v /" | python -c "import sys,json; l=sys.stdin.read(); v,j=l.split(' ',1); d=json.loads(j); print(v, 'cfg5', d['graph_ms'], d['stages_us'])"
done
done
