python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/tmem_occ tools/tmem_occ_probe.cu && timeout 60 /tmp/tmem_occ
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numerics.py tests/test_gpu_sweep.py -q -m gpu -x 2>&1 | tail -2
for W in G Q A R L; do echo "== $W"; timeout 300 python tools/trace_one.py $W best tools/data/best_r32.json 2>&1 | head -${TRACE_LINES:-22} | cut -c1-200; done
