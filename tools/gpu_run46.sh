python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 120 python tools/trace_one.py A "Kt.3.i,O.3.x,V.2.i,V.3.x" '{"x":128,"i":8192}' 2>&1 | head -4 | cut -c1-150
timeout 120 python tools/trace_one.py A "Kt.3.i,O.3.x,V.2.i,V.3.x" '{"x":64,"i":4096}' 2>&1 | head -4 | cut -c1-150
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numerics.py tests/test_gpu_sweep.py -q -m gpu -x 2>&1 | tail -2
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -3 gpurun_out/bench.err
