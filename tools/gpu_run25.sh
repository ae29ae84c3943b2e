python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
for U in none 1 2; do
  if [ $U = none ]; then unset SGM_EW_UNROLL; else export SGM_EW_UNROLL=$U; fi
  echo "== G unroll=$U"; timeout 300 python tools/trace_one.py G best tools/data/best_r21.json 2>&1 | head -24 | cut -c1-200
  echo "== Q unroll=$U"; timeout 300 python tools/trace_one.py Q best tools/data/best_r21.json 2>&1 | head -24 | cut -c1-200
done
