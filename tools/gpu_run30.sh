python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/pytest_gpu.log
for P in 0 1; do
  if [ $P = 1 ]; then export SGM_NO_PDL=1; else unset SGM_NO_PDL; fi
  for W in G Q A R L; do echo "== $W nopdl=$P"; timeout 300 python tools/trace_one.py $W best tools/data/best_r29.json 2>&1 | head -${TRACE_LINES:-14} | cut -c1-200; done
done
