set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python tools/diag_candidates.py G > gpurun_out/diag_G.log 2>&1; cat gpurun_out/diag_G.log | cut -c1-300
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --records gpurun_out/records.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -8 gpurun_out/bench.err; cat gpurun_out/bench.json
