"""One launch each of the c4 hot kernels at their bench shapes (for ncu)."""
import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2602_10016_b200._capi import gemm
from paper_2602_10016_b200 import functional as F, attention as A
from paper_2602_10016_b200.tensor import Params
torch.manual_seed(0)
B, T, d, H = 32, 4096, 512, 8
S = (torch.randn(B * T, d, device="cuda") / 22).bfloat16()
W = (torch.randn(3 * d, d, device="cuda") / 22).bfloat16()
what = sys.argv[1] if len(sys.argv) > 1 else "all"
for _ in range(2):
    if what in ("all", "gemm"):
        qkv = gemm(S, W.t())                     # QKV projection fwd (M=131072, N=1536, K=512)
    if what in ("all", "swa"):
        qkv3 = gemm(S, W.t()).view(B, T, 3 * d)
        lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
        q = qkv3.detach().requires_grad_()
        o = F.swa_core(q, lens, H, 64, 128, False)
        o.backward(torch.randn_like(o))
    torch.cuda.synchronize()
print("ok")
