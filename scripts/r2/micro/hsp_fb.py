"""HSP pooling d=512 fwd + bwd (functional, c4 shape) timing: kl_hsp_fwd / kl_hsp_bwd only (CUDA events around the calls)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
from paper_2602_10016_b200 import functional as F
_capi.lib()
import os
B, T, d, HQ = [int(x) for x in os.environ.get("SHAPE", "32,4096,512,320").split(",")]
torch.manual_seed(0)
S = (torch.randn(B, T, d, device="cuda") / 22).bfloat16().requires_grad_()
Q = (torch.randn(HQ, d, device="cuda") / 22).requires_grad_()
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
n1 = HQ * 4 // 5
g1 = torch.randn(B, n1, d, device="cuda").bfloat16(); g2 = torch.randn(B, HQ - n1, d, device="cuda").bfloat16()
for _ in range(3):
    o1, o2 = F.hsp_pool(S, Q, lens, splits=(n1, HQ - n1)); torch.autograd.backward([o1, o2], [g1, g2])
torch.cuda.synchronize()
_capi.TIMED = {"kl_hsp_fwd": [], "kl_hsp_bwd": []}
for _ in range(10):
    o1, o2 = F.hsp_pool(S, Q, lens, splits=(n1, HQ - n1)); torch.autograd.backward([o1, o2], [g1, g2])
torch.cuda.synchronize()
for k, v in _capi.TIMED.items():
    print(k, f"{sum(s.elapsed_time(e) for s, e in v) / len(v) * 1e3:.1f} us")
