"""GDPA core d=512 fwd + bwd (functional, c4 shape) timing of kl_gdpa_fwd / kl_gdpa_bwd."""
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
from paper_2602_10016_b200 import functional as F
_capi.lib()
B, T, d = 32, 4096, 512
torch.manual_seed(0)
S = (torch.randn(B, T, d, device="cuda") / 22).bfloat16().requires_grad_()
Kt = (torch.randn(B, 128, d, device="cuda") / 2).bfloat16().requires_grad_()
Vt = (torch.randn(B, 128, d, device="cuda") / 8).bfloat16().requires_grad_()
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
g = torch.randn(B, T, d, device="cuda").bfloat16()
acts = ("silu", "relu", "identity", "tanh") * 2
for _ in range(3):
    y = F.gdpa_core(S, Kt, Vt, lens, acts, 16, 1.0 / T); y.backward(g)
torch.cuda.synchronize()
_capi.TIMED = {"kl_gdpa_fwd": [], "kl_gdpa_bwd": []}
for _ in range(10):
    y = F.gdpa_core(S, Kt, Vt, lens, acts, 16, 1.0 / T); y.backward(g)
torch.cuda.synchronize()
for k, v in _capi.TIMED.items():
    print(k, f"{sum(s.elapsed_time(e) for s, e in v) / len(v) * 1e3:.1f} us")
