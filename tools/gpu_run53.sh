python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_numerics.py tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
echo "== L"; timeout 120 python tools/trace_one.py L best tools/data/best_r49.json 2>&1 | head -12 | cut -c1-160
timeout 900 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --best-out gpurun_out/best.json > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -2 gpurun_out/bench.err
python -c "
import json; b=json.load(open('gpurun_out/best.json'))
for w,x in b.items(): print(w, '%.2f us'%x['latency_us'], '%.0f%%'%(100*x['frac_hbm']), x['template'], x['hints'], x['plan'][:110])
"
