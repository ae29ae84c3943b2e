python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numerics.py tests/test_gpu_sweep.py -q -m gpu -x 2>&1 | tail -2
for W in G L A R Q; do python tools/pdl_probe.py $W tools/data/best_r29.json; SGM_NO_PDL=1 python tools/pdl_probe.py $W tools/data/best_r29.json; done
for W in G Q A R L; do echo "== $W"; timeout 300 python tools/trace_one.py $W best tools/data/best_r29.json 2>&1 | head -${TRACE_LINES:-16} | cut -c1-200; done
