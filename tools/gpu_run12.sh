python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -8 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --records gpurun_out/records.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -3 gpurun_out/bench.err
python tools/best.py gpurun_out/records.json 2
for W in A G L; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof12_$W python tools/profile_one.py $W best gpurun_out/records.json --iters 8 > gpurun_out/ncu12_$W.log 2>&1; echo "ncu $W rc $?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:sgm_cand --csv --log-file gpurun_out/launch12_$W.csv python tools/profile_one.py $W best gpurun_out/records.json --iters 20 > /dev/null 2>&1
done
