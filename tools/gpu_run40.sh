python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc $?"; tail -3 gpurun_out/smoke.log
S=$(date +%s); timeout 1500 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench default rc $? in $(( $(date +%s) - S ))s"; tail -2 gpurun_out/bench_default.err; head -c 600 gpurun_out/bench_default.json; echo
S=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "bench ref rc $? in $(( $(date +%s) - S ))s"; head -c 400 gpurun_out/bench_ref.json; echo
for W in G A Q L R; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof40_$W python tools/profile_one.py $W best tools/data/best_r39.json --iters 8 > gpurun_out/ncu40_$W.log 2>&1; echo "ncu $W rc $?"
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches40_G.csv python bench.py --workloads G --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --tune-top 1 --best-iters 20 > gpurun_out/launch_bench.json 2>&1; echo "ncu list rc $?"
