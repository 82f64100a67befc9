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
    elif which.startswith("mlp"):  # Wukong expert MLP layer 0 (B * n_i = 3072 rows, d -> 2d)
        x = S.view(-1, d)[:3072]
        W0 = torch.randn(2 * d, d, device="cuda", generator=g).to(bf)
        b0 = torch.randn(2 * d, device="cuda", generator=g)
        y = torch.empty(3072, 2 * d, device="cuda", dtype=bf)
        pre = torch.empty_like(y)
        if which == "mlp":
            gemm(x, W0.t(), y, bias=b0, acts=["silu"], aux=pre, aux_mode=1)
        elif which == "mlp_noaux":
            gemm(x, W0.t(), y, bias=b0, acts=["silu"])
        elif which == "mlp_bias":
            gemm(x, W0.t(), y, bias=b0)
        else:
            gemm(x, W0.t(), y)
    elif which == "dx":  # attention-input gradient: dQKV @ Wqkv, accumulated onto the residual gradient
        gemm(out3, W, out1, residual=out1)
    else:
        gemm(S, W[:d].t(), out1, residual=S)
torch.cuda.synchronize()
