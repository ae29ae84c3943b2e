python -c "from paper_2604_15272_b200 import build as B; B.build_lib()" > gpurun_out/build.log 2>&1
python - <<'PY'
import torch
x=torch.empty(235_000_000//2, dtype=torch.bfloat16, device='cuda'); y=torch.empty_like(x)
for _ in range(3): y.copy_(x)
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20): y.copy_(x)
e1.record(); torch.cuda.synchronize()
print("torch copy 235MB: %.1f us, %.0f GB/s (r+w)"%(e0.elapsed_time(e1)/20*1e3, 2*235e6/(e0.elapsed_time(e1)/20*1e-3)/1e9))
s=x.float() if False else None
PY
for MC in 1 2 4 8; do for X in 8 16 32 64 128; do
timeout 120 python tools/gemv_probe.py bf16 8 4096 14336 $X "{\"max_cluster\":$MC}" 2>&1 | tail -1 | cut -c1-260
done; done
for MC in 1 4 8; do for X in 16 64 128 256; do
timeout 120 python tools/gemv_probe.py f32 8 4096 4096 $X "{\"max_cluster\":$MC}" 2>&1 | tail -1 | cut -c1-260
done; done
for T in 128 256 512; do
timeout 120 python tools/gemv_probe.py bf16 8 4096 14336 16 "{\"max_cluster\":1,\"threads\":$T}" 2>&1 | tail -1 | cut -c1-260
done
timeout 120 python tools/gemv_probe.py bf16 8 4096 14336 16 '{"max_cluster":1, "target_ctas": 148}' 2>&1 | tail -1 | cut -c1-260
timeout 120 python tools/gemv_probe.py bf16 8 4096 14336 16 '{"max_cluster":1, "target_ctas": 1024}' 2>&1 | tail -1 | cut -c1-260
timeout 120 python tools/gemv_probe.py bf16 8 4096 14336 16 '{"max_cluster":1, "no_tma": 1}' 2>&1 | tail -1 | cut -c1-260
timeout 120 python tools/gemv_probe.py bf16 8 4096 14336 16 '{"max_cluster":1, "use_tcgen05": -1}' 2>&1 | tail -1 | cut -c1-260
