python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -4 gpurun_out/pytest_gpu.log
timeout 120 python tools/trace_one.py R best tools/data/best_r35.json 2>&1 | head -16 | cut -c1-200
for H in '{"one_cta":1}' '{}'; do timeout 120 python tools/gemv_probe.py f32 8 4096 4096 32 "$H" | cut -c1-200; done
timeout 1500 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --records gpurun_out/records.json --best-out gpurun_out/best.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -3 gpurun_out/bench.err
python -c "
import json; b=json.load(open('gpurun_out/best.json'))
for w,x in b.items(): print(w, '%.2f us'%x['latency_us'], '%.0f%%'%(100*x['frac_hbm']), x['template'], x['hints'], x['params'], x['mapping'], x['plan'][:150])
"
