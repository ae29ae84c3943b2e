python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for W in A G; do echo "== $W"; timeout 120 python tools/trace_one.py $W best tools/data/best_r39.json 2>&1 | head -22 | cut -c1-160; echo "== $W dup"; SGM_DUP_EW=1 timeout 120 python tools/trace_one.py $W best tools/data/best_r39.json 2>&1 | head -22 | cut -c1-160; done
