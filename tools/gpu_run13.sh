python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/check_one.py A "Kt.2.i,O.3.x,Q.3.i,V.3.x" '{"x":2,"i":16}' '[{}, {"no_tma":1}, {"max_cluster":8}, {"no_hoist":1}]' 2>&1 | tail -20
timeout 1200 python -m pytest tests -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -8 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --records gpurun_out/records.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -3 gpurun_out/bench.err
python tools/best.py gpurun_out/records.json 2
for W in L A Q; do timeout 300 python tools/trace_one.py $W best gpurun_out/records.json 2>&1 | head -22 | cut -c1-200; done
