"""c2 projection GEMMs (d = 256, K = 256 / 768): ours (batched over 128 samples as the model
calls them, and flat) vs cuBLAS, with GBs of HBM traffic per call for the roofline."""
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
_capi.lib()
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for name, Bn, M, N, K in (("qkv fwd", 128, 1024, 768, 256), ("out fwd", 128, 1024, 256, 256),
                          ("qkv dX", 128, 1024, 256, 768)):
    A = (torch.randn(Bn, M, K, device="cuda") / 16).bfloat16()
    W = (torch.randn(N, K, device="cuda") / 16).bfloat16()
    out = torch.empty(Bn, M, N, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: _capi.gemm(A, W.t(), out))
    msf = t(lambda: _capi.gemm(A.view(Bn * M, K), W.t(), out.view(Bn * M, N)))
    msc = t(lambda: torch.matmul(A.view(Bn * M, K), W.t(), out=out.view(Bn * M, N)))
    gb = (Bn * M * K + Bn * M * N) * 2 / 1e9
    print(f"{name:8s} batched {ms*1e3:6.1f} us ({gb/ms*1e-3*1e3:5.2f} TB/s) | flat {msf*1e3:6.1f} us | cublas {msc*1e3:6.1f} us"
          f" ({gb/msc:5.2f} TB/s)", flush=True)
