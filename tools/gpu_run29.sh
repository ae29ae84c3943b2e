python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --steps 2 --warmup 3 --records gpurun_out/records.json --best-out gpurun_out/best.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -4 gpurun_out/bench.err; cat gpurun_out/bench.json | head -c 1500; echo
python -c "
import json; b=json.load(open('gpurun_out/best.json'))
for w,x in b.items(): print(w, '%.2f us'%x['latency_us'], '%.0f%%'%(100*x['frac_hbm']), x['template'], x['hints'], x['params'], x['mapping'], x['plan'][:150])
"
for W in G R A Q L; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof29_$W python tools/profile_one.py $W best gpurun_out/best.json --iters 8 > gpurun_out/ncu29_$W.log 2>&1; echo "ncu $W rc $?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches29_G.csv python bench.py --workloads G --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --tune-top 1 --best-iters 20 > gpurun_out/launch_bench.json 2>&1; echo "ncu list rc $?"
for W in G Q A R L; do echo "== $W"; timeout 300 python tools/trace_one.py $W best gpurun_out/best.json 2>&1 | head -26 | cut -c1-200; done
