python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for v in 0 1 2 3 4; do export SGM_CLB=$v
for W in G R; do echo "== $W clb=$v"; timeout 300 python tools/trace_one.py $W best tools/data/best_r21.json 2>&1 | head -14 | cut -c1-200; done; done
