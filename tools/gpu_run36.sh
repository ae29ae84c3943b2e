python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for H in '{}' '{"one_cta":1}' '{"max_cluster":1}' '{"one_cta":1,"max_cluster":1}'; do
  timeout 120 python tools/gemv_probe.py f32 8 4096 4096 32 "$H" | cut -c1-220
  timeout 120 python tools/gemv_probe.py bf16 8 4096 4096 32 "$H" | cut -c1-220
done
timeout 120 python tools/gemv_probe.py f32 8 4096 4096 32 '{"one_cta":1}' --trace | cut -c1-200
timeout 120 python tools/trace_one.py R best tools/data/best_r35.json 2>&1 | head -40 | cut -c1-200
for W in G A Q L R; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sgm_cand -s 5 -c 1 -o gpurun_out/prof36_$W python tools/profile_one.py $W best tools/data/best_r35.json --iters 8 > gpurun_out/ncu36_$W.log 2>&1; echo "ncu $W rc $?"
done
