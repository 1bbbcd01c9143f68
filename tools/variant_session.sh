python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
bash tools/build_variants.sh ys4 "-DIBK_YSTAGES=4" ys5 "-DIBK_YSTAGES=5" ys6 "-DIBK_YSTAGES=6" > /dev/null 2>&1
for rep in 1 2; do
for v in default ys4 ys5 ys6; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 4 30 2>/dev/null | sed "s/^/$v /" | python -c "import sys,json; l=sys.stdin.read(); v,j=l.split(' ',1); d=json.loads(j); print(v, d['graph_ms'], d['stages_us']['y_fwd'], d['stages_us']['y_inv'])"
done
done
for v in default ys4 ys6; do
  if [ $v = default ]; then L=""; else L="build_variants/$v.so"; fi
  IB_B200_LIB=$L python tools/stage_bench_cfg.py 5 8 2>/dev/null | sed "s/^/$v /" | python -c "import sys,json; l=sys.stdin.read(); v,j=l.split(' ',1); d=json.loads(j); print(v, 'cfg5', d['graph_ms'], d['stages_us']['y_fwd'], d['stages_us']['y_inv'])"
done
