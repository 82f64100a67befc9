import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200._capi import gemm, lib
torch.manual_seed(0)
for (M, N, K) in [(8192, 192, 64), (4096, 192, 64), (8192, 128, 64), (8192, 256, 64), (8192, 192, 128), (16384, 192, 64), (8192, 64, 64), (6144, 192, 64), (8320, 192, 64)]:
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(N, K, device="cuda").bfloat16()
    ref = A.float() @ W.float().t()
    for trial in range(2):
        out = torch.full((M, N), float("nan"), device="cuda", dtype=torch.bfloat16) if trial else None
        c = gemm(A, W.t(), out)
        torch.cuda.synchronize()
        err = ((c.float() - ref).abs().max() / ref.abs().max()).item()
        nbad = int((~torch.isfinite(c.float())).sum())
        rows = (~torch.isfinite(c.float())).any(1).nonzero().flatten()
        print(M, N, K, "prefill-nan" if trial else "empty", "err", f"{err:.2e}", "nonfinite", nbad, "rows", rows[:4].tolist(), rows[-2:].tolist() if len(rows) else [])
