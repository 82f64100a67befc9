import sys, os, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200._capi import gemm
torch.manual_seed(0)
bn = os.environ.get("KL_GEMM_BN", "auto")
for (M, N, K) in [(8192, 192, 64), (16384, 192, 64), (8192, 160, 64), (8192, 224, 64), (8192, 96, 64), (20000, 192, 64), (8192, 384, 64)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(N, K, device="cuda").bfloat16()
    ref = A.float() @ W.float().t()
    bad = 0
    for trial in range(3):
        c = gemm(A, W.t())
        torch.cuda.synchronize()
        bad += int((~torch.isfinite(c.float())).sum()) + int(((c.float() - ref).abs() > 0.05 * ref.abs().max()).sum())
    print("BN", bn, M, N, K, "bad", bad)
