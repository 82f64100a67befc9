"""Isolated timing of the c4 weight-gradient GEMM shapes (fp32 accumulate into a flat buffer)."""
import sys
import torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
_capi.lib()
torch.manual_seed(0)
for name, M, N, K in (("qkv dW", 1536, 512, 131072), ("out dW", 512, 512, 131072), ("c2 qkv dW", 768, 256, 131072)):
    A = torch.randn(K, M, device="cuda").bfloat16()   # dY (K rows) -> A = dY^T (MN-major)
    Bm = torch.randn(K, N, device="cuda").bfloat16()
    C = torch.zeros(M, N, device="cuda")
    for _ in range(3):
        _capi.gemm(A.t(), Bm, C, beta=1.0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        _capi.gemm(A.t(), Bm, C, beta=1.0)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    C2 = torch.zeros(M, N, device="cuda"); _capi.gemm(A.t(), Bm, C2, beta=1.0)
    ref = (A.t().float() @ Bm.float())
    err = ((C2 - ref).norm() / ref.norm()).item()
    print(f"{name}: {ms * 1e3:7.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TF/s  rel err {err:.2e}")
