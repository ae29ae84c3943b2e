# usage: bash tools/gpu_trace.sh <best.json> [pytest-files...]  (traces G Q A R L)
B=$1; shift
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ $# -gt 0 ]; then timeout 900 python -m pytest "$@" -q -m gpu -x 2>&1 | tail -2; fi
for W in G Q A R L; do echo "== $W"; timeout 300 python tools/trace_one.py $W best $B 2>&1 | head -${TRACE_LINES:-24} | cut -c1-200; done
