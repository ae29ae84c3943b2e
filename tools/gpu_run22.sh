python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_numerics.py -q -m gpu -x > gpurun_out/pytest_num.log 2>&1; echo "pytest rc $?"; tail -2 gpurun_out/pytest_num.log
for W in G A L R Q; do
  for E in 0 1; do
    if [ $E = 1 ]; then export SGM_LATE_STREAM=1; else unset SGM_LATE_STREAM; fi
    echo "== $W early=$E"
    timeout 300 python tools/trace_one.py $W best tools/data/best_r21.json 2>&1 | cut -c1-200
  done
done
