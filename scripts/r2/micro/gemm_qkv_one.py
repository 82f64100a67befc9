"""One c4 QKV-projection GEMM (131072 x 1536 x 512) by ours and by cuBLAS (comparison under ncu)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
_capi.lib()
M, N, K = 131072, 1536, 512
A = (torch.randn(M, K, device="cuda") / 22).bfloat16()
W = (torch.randn(N, K, device="cuda") / 22).bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    _capi.gemm(A, W.t(), out)
    torch.matmul(A, W.t(), out=out)
torch.cuda.synchronize()
