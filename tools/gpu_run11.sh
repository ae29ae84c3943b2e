python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -25 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --records gpurun_out/records.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -4 gpurun_out/bench.err
python /root/repo/tools/best.py gpurun_out/records.json 3 2>/dev/null
for W in G A R Q L; do timeout 300 python tools/trace_one.py $W best gpurun_out/records.json 2>&1 | head -14 | cut -c1-200; done
