"""One launch each of the c4 hot kernels at their bench shapes (B = 32,
T = 4096, d = 512, H = 8) for ncu: the QKV projection GEMM, the banded
attention forward / backward, the fused GDPA and HSP kernels (d = 512) and
one Adam range.  Usage: prof_kernels.py [gemm|swa|gdpa|hsp|adam|all]"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200 import functional as F  # noqa: E402
from paper_2602_10016_b200._capi import gemm  # noqa: E402

torch.manual_seed(0)
B, T, d, H = 32, 4096, 512, 8
what = sys.argv[1] if len(sys.argv) > 1 else "all"
S = (torch.randn(B * T, d, device="cuda") / 22).bfloat16()
lens = torch.full((B,), T, dtype=torch.int32, device="cuda")
for _ in range(2):
    if what in ("all", "gemm"):
        W = (torch.randn(3 * d, d, device="cuda") / 22).bfloat16()
        gemm(S, W.t())  # QKV projection fwd (M = 131072, N = 1536, K = 512)
    if what in ("all", "swa"):
        W = (torch.randn(3 * d, d, device="cuda") / 22).bfloat16()
        q = gemm(S, W.t()).view(B, T, 3 * d).detach().requires_grad_()
        o = F.swa_core(q, lens, H, 64, 128, False)
        o.backward(torch.randn_like(o))
    if what in ("all", "gdpa"):
        S3 = S.view(B, T, d).detach().requires_grad_()
        Kt = (torch.randn(B, 128, d, device="cuda") / 2).bfloat16().requires_grad_()
        Vt = (torch.randn(B, 128, d, device="cuda") / 8).bfloat16().requires_grad_()
        y = F.gdpa_core(S3, Kt, Vt, lens, ("silu", "relu", "identity", "tanh") * 2, 16, 1.0 / T)
        y.backward(torch.randn_like(y))
    if what in ("all", "hsp"):
        S3 = S.view(B, T, d).detach().requires_grad_()
        Q = (torch.randn(320, d, device="cuda") / 22).requires_grad_()
        o1, o2 = F.hsp_pool(S3, Q, lens, splits=(256, 64))
        torch.autograd.backward([o1, o2], [torch.randn_like(o1), torch.randn_like(o2)])
    if what in ("all", "adam"):
        from paper_2602_10016_b200 import _capi
        n = 40_000_000
        p = torch.zeros(n, device="cuda"); g = torch.randn(n, device="cuda") * 1e-3
        m = torch.zeros(n, device="cuda"); v = torch.zeros(n, device="cuda")
        wc = torch.empty(n, device="cuda", dtype=torch.bfloat16); t = torch.zeros(1, dtype=torch.int32, device="cuda")
        _capi.call("kl_adam_step", n, 1e-3, 0.9, 0.999, 1e-8, 0, t.data_ptr(), p.data_ptr(), g.data_ptr(),
                   m.data_ptr(), v.data_ptr(), wc.data_ptr(), _capi._stream())
    torch.cuda.synchronize()
print("ok")
