python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
echo "== G"; timeout 300 python tools/trace_one.py G best tools/data/best_r21.json 2>&1 | cut -c1-200
echo "== G cl1"; timeout 300 python tools/trace_one.py G best tools/data/best_r21.json '{"max_cluster":1}' 2>&1 | cut -c1-200
echo "== Q"; timeout 300 python tools/trace_one.py Q best tools/data/best_r21.json 2>&1 | cut -c1-200
