python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1400 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -2 gpurun_out/smoke.log
S=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc $? in $(( $(date +%s) - S ))s"; tail -3 gpurun_out/bench_default.err
python -c "
import json; d=json.load(open('gpurun_out/bench_default.json'))
print({k:d[k] for k in ['value','e2e','roofline','cpu_baseline','clocks','gpu_launches'] if k in d})
for w,x in d['best_kernels'].items(): print(w, round(x['latency_us'],2), round(x['frac_hbm'],3), x['hints'])
"
