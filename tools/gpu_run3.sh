set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_numerics.py -x -q > gpurun_out/pytest_num.log 2>&1; echo "num rc $?"; tail -15 gpurun_out/pytest_num.log
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc $?"; tail -15 gpurun_out/pytest_gpu.log
timeout 1200 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline --records gpurun_out/records.json > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc $?"
tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
