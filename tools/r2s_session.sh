python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
mkdir -p gpurun_out
python tools/prof_step.py --config 4 --warmup 2 --steps 1 > /dev/null 2>&1
NL=$(ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_step.py --config 4 --warmup 2 --steps 1 2>/dev/null | grep -c gpu__time_duration)
echo "launches $NL"
timeout 900 ncu --set full --clock-control none --import-source on -s $((NL - 9)) -c 9 -o gpurun_out/prof_r2s python tools/prof_step.py --config 4 --warmup 2 --steps 1 > gpurun_out/ncu_r2s.log 2>&1; echo "ncu rc=$?"
ls -la gpurun_out/prof_r2s.ncu-rep
