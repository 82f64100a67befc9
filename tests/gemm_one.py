"""Run one model-shaped kl_gemm a few times (for ncu)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200._capi import gemm  # noqa: E402

which = sys.argv[1]
g = torch.Generator(device="cuda").manual_seed(0)
bf = torch.bfloat16
B, T, d = 128, 1024, 256
S = torch.randn(B, T, d, device="cuda", generator=g).to(bf)
W = torch.randn(3 * d, d, device="cuda", generator=g).to(bf)
bias = torch.randn(d, device="cuda", generator=g)
out3 = torch.empty(B, T, 3 * d, device="cuda", dtype=bf)
out1 = torch.empty(B, T, d, device="cuda", dtype=bf)
for _ in range(3):
    if which == "qkv":
        gemm(S, W.t(), out3)
    elif which == "bias":
        gemm(S, W[:d].t(), out1, bias=bias)
    elif which == "dx":  # attention-input gradient: dQKV @ Wqkv, accumulated onto the residual gradient
        gemm(out3, W, out1, residual=out1)
    else:
        gemm(S, W[:d].t(), out1, residual=S)
torch.cuda.synchronize()
