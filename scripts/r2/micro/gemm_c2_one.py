"""One c2 output-projection GEMM (128 x 1024 x 256 x 256, bf16) for ncu."""
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
A = (torch.randn(128, 1024, 256, device="cuda") / 16).bfloat16()
W = (torch.randn(256, 256, device="cuda") / 16).bfloat16()
out = torch.empty(128, 1024, 256, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    _capi.gemm(A, W.t(), out)
    torch.matmul(A.view(-1, 256), W.t(), out=out.view(-1, 256))
torch.cuda.synchronize()
