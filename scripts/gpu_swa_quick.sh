timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "swa or model" 2>&1 | tail -1
timeout 300 python scripts/probes/swa_tc_probe.py bwd_only 128 1024 4 128 0 full > /dev/null 2>&1
timeout 300 python - <<'PY'
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import functional as F
B, T, H, dh, w = 128, 1024, 4, 64, 128
qkv = torch.randn(B, T, 3 * H * dh, device="cuda").to(torch.bfloat16).requires_grad_()
lens = torch.full((B,), T, device="cuda", dtype=torch.int32)
go = torch.randn(B, T, H * dh, device="cuda").to(torch.bfloat16)
for _ in range(3):
    o = F.swa_core(qkv, lens, H, dh, w); o.backward(go)
torch.cuda.synchronize()
e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
e[0].record()
for _ in range(10): o = F.swa_core(qkv, lens, H, dh, w)
e[1].record()
for _ in range(10): o.backward(go, retain_graph=True)
e[2].record(); torch.cuda.synchronize()
fwd = e[0].elapsed_time(e[1]) / 10; bwd = e[1].elapsed_time(e[2]) / 10
fl = 4.0 * B * H * dh * sum(min(i + w, T - 1) - max(i - w, 0) + 1 for i in range(T))
print(f"swa fwd {fwd*1e3:.1f} us ({fl/fwd/1e9:.0f} TF/s)  bwd {bwd*1e3:.1f} us ({2.5*fl/bwd/1e9:.0f} TF/s)")
PY
