import sys, os, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200._capi import gemm
torch.manual_seed(0)
shapes = [("qkv_fwd", 131072, 1536, 512), ("out_fwd", 131072, 512, 512), ("qkv_dx", 131072, 512, 1536)]
for name, M, N, K in shapes:
    A = (torch.randn(M, K, device="cuda") / 22).bfloat16()
    W = (torch.randn(N, K, device="cuda") / 22).bfloat16()
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(3): gemm(A, W.t(), out)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20): gemm(A, W.t(), out)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(os.environ.get("KL_GEMM_BN", "auto"), name, f"{ms*1e3:.1f} us", f"{2*M*N*K/ms/1e9:.0f} TF/s")
