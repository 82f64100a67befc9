"""Our tcgen05 GEMM vs torch.matmul (cuBLAS) on the c4 projection shapes (comparison only)."""
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
for name, M, N, K in (("qkv fwd", 131072, 1536, 512), ("out fwd", 131072, 512, 512), ("qkv dX", 131072, 512, 1536),
                      ("sq 8192", 8192, 8192, 8192), ("hsp 640", 131072, 512, 640)):
    A = (torch.randn(M, K, device="cuda") / 22).bfloat16()
    W = (torch.randn(N, K, device="cuda") / 22).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: _capi.gemm(A, W.t(), out))
    msc = t(lambda: torch.matmul(A, W.t(), out=out))
    f = 2 * M * N * K
    print(f"{name:8s} ours {ms*1e3:7.1f} us {f/ms/1e9:6.0f} TF/s | cublas {msc*1e3:7.1f} us {f/msc/1e9:6.0f} TF/s", flush=True)
for name, M, N, K in (("qkv dW", 1536, 512, 131072), ("out dW", 512, 512, 131072)):
    A = torch.randn(K, M, device="cuda").bfloat16()
    Bm = torch.randn(K, N, device="cuda").bfloat16()
    C = torch.zeros(M, N, device="cuda")
    ms = t(lambda: _capi.gemm(A.t(), Bm, C, beta=1.0))
    Cb = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    msc = t(lambda: torch.matmul(A.t(), Bm, out=Cb))
    f = 2 * M * N * K
    print(f"{name:8s} ours {ms*1e3:7.1f} us {f/ms/1e9:6.0f} TF/s | cublas(bf16 out) {msc*1e3:7.1f} us {f/msc/1e9:6.0f} TF/s", flush=True)
# operand-major experiments: square with MN-major A; dW with K-major (transposed copies)
M = N = K = 8192
A = (torch.randn(K, M, device="cuda") / 90).bfloat16()
W = (torch.randn(N, K, device="cuda") / 90).bfloat16()
out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
ms = t(lambda: _capi.gemm(A.t(), W.t(), out)); print(f"sq MN-major A  ours {2*M*N*K/ms/1e9:6.0f} TF/s")
C = torch.zeros(M, N, device="cuda")
ms = t(lambda: _capi.gemm(A.t(), W.t(), C, beta=1.0)); print(f"sq MN-major A fp32 acc ours {2*M*N*K/ms/1e9:6.0f} TF/s")
for name, M, N, K in (("qkv dW Kmaj", 1536, 512, 131072),):
    A = torch.randn(M, K, device="cuda").bfloat16()
    Bm = torch.randn(N, K, device="cuda").bfloat16()
    C = torch.zeros(M, N, device="cuda")
    ms = t(lambda: _capi.gemm(A, Bm.t(), C, beta=1.0)); print(f"{name} fp32 acc ours {2*M*N*K/ms/1e9:6.0f} TF/s")
    Cb = torch.zeros(M, N, device="cuda", dtype=torch.bfloat16)
    ms = t(lambda: _capi.gemm(A, Bm.t(), Cb)); print(f"{name} bf16 out ours {2*M*N*K/ms/1e9:6.0f} TF/s")
