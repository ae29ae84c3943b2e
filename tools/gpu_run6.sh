set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1200 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --records gpurun_out/records.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -8 gpurun_out/bench.err; cat gpurun_out/bench.json
for W in G A; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof6_$W python tools/profile_one.py $W best gpurun_out/records.json --iters 8 > gpurun_out/ncu6_$W.log 2>&1; echo "ncu $W rc $?"
done
