set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python bench.py --steps 2 --warmup 3 --records gpurun_out/records.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_G.csv python bench.py --workloads G --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --budget-us 200 > gpurun_out/ncu_bench_G.log 2>&1; echo "ncu list rc $?"
for W in G R A Q L; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof_$W python tools/profile_one.py $W best gpurun_out/records.json --iters 8 > gpurun_out/ncu_$W.log 2>&1; echo "ncu $W rc $?"
done
ls -la gpurun_out
