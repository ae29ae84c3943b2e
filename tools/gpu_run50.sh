python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for W in G R A Q L; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof50_$W python tools/profile_one.py $W best tools/data/best_r49.json --iters 8 > gpurun_out/ncu50_$W.log 2>&1; echo "ncu $W rc $?"
done
for W in G R; do echo "== $W"; timeout 120 python tools/trace_one.py $W best tools/data/best_r49.json 2>&1 | head -20 | cut -c1-160; done
