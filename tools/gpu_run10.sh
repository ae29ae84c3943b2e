python -c "from paper_2604_15272_b200 import build as B; B.build_lib()" > gpurun_out/build.log 2>&1
for MC in 2 4 8; do for X in 8 128; do
timeout 120 python tools/gemv_probe.py bf16 8 4096 14336 $X "{\"max_cluster\":$MC}" 2>&1 | tail -1 | cut -c1-230
done; done
for MC in 4 8; do for X in 64 128; do
timeout 120 python tools/gemv_probe.py f32 8 4096 4096 $X "{\"max_cluster\":$MC}" 2>&1 | tail -1 | cut -c1-230
done; done
R=profiles/records/r01c_top20.json
for W in G A; do timeout 300 python tools/trace_one.py $W best $R 2>&1 | head -12 | cut -c1-200; done
