"""dW shape (1536 x 512, K = 131072) with each operand-major combination (fp32 accumulate)."""
import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
_capi.lib()
def t(fn, n=10):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for (M, N) in ((1536, 512), (512, 512)):
    K = 131072
    f = 2 * M * N * K
    Ak = torch.randn(M, K, device="cuda").bfloat16(); Am = Ak.t().contiguous().t()   # Am: MN-major view
    Bk = torch.randn(N, K, device="cuda").bfloat16().t(); Bm = Bk.contiguous()       # Bk (K,N) K-major view; Bm row-major (MN-major)
    C = torch.zeros(M, N, device="cuda")
    for an, A in (("A K", Ak), ("A MN", Am)):
        for bn, B in (("B K", Bk), ("B MN", Bm)):
            ms = t(lambda: _capi.gemm(A, B, C, beta=1.0))
            print(f"{M}x{N} {an:5s} {bn:5s} {ms*1e3:7.1f} us {f/ms/1e9:6.0f} TF/s", flush=True)
    # batched-reduced form like the model's (b x 4096 rows)
    A3 = Am.t().reshape(32, 4096, M)   # (b, k, M) contiguous -> A[b] = A3[b].t() MN-major
    B3 = Bm.reshape(32, 4096, N)
    ms = t(lambda: _capi.gemm(A3.transpose(1, 2), B3, C, beta=1.0, reduce=(False, True)))
    print(f"{M}x{N} batched-reduced MN/MN {ms*1e3:7.1f} us {f/ms/1e9:6.0f} TF/s", flush=True)
