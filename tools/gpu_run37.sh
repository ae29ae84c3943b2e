python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_numerics.py -q -m gpu -x 2>&1 | tail -2
for H in '{"one_cta":1}' '{"one_cta":1,"max_cluster":1}' '{}'; do timeout 120 python tools/gemv_probe.py f32 8 4096 4096 32 "$H" | cut -c1-200; done
timeout 120 python tools/trace_one.py R best tools/data/best_r35.json 2>&1 | head -12 | cut -c1-200
