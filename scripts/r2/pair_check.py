import sys, os, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200._capi import gemm
torch.manual_seed(0)
ok = True
cases = [(512, 256, 64, "kk"), (131072 // 16, 1536, 512, "kk"), (8192, 512, 1536, "kn"), (1000, 384, 200, "kk"),
         (4096, 256, 4096, "mn")]
for M, N, K, lay in cases:
    A = (torch.randn(M, K, device="cuda") / 8).bfloat16()
    if lay == "kk":
        W = (torch.randn(N, K, device="cuda") / 8).bfloat16(); Bm = W.t()
    elif lay == "kn":
        Bm = (torch.randn(K, N, device="cuda") / 8).bfloat16()
    else:  # MN-major A
        A = (torch.randn(K, M, device="cuda") / 8).bfloat16().t(); Bm = (torch.randn(K, N, device="cuda") / 8).bfloat16()
    ref = A.double() @ Bm.double()
    c = gemm(A, Bm)
    torch.cuda.synchronize()
    err = ((c.double() - ref).abs().max() / ref.abs().max()).item()
    fin = bool(torch.isfinite(c).all())
    R = torch.randn(M, N, device="cuda").bfloat16()
    c2 = gemm(A, Bm, residual=R)
    torch.cuda.synchronize()
    err2 = ((c2.double() - ref - R.double()).abs().max() / ref.abs().max()).item()
    c3 = torch.zeros(M, N, device="cuda")
    gemm(A, Bm, c3, beta=1.0)
    gemm(A, Bm, c3, beta=1.0)
    torch.cuda.synchronize()
    err3 = ((c3.double() - 2 * ref).abs().max() / (2 * ref).abs().max()).item()
    print(M, N, K, lay, "err", f"{err:.2e}", "res", f"{err2:.2e}", "acc32", f"{err3:.2e}", "finite", fin, flush=True)
    ok &= err < 1e-2 and err2 < 1e-2 and err3 < 1e-2 and fin
print("PASS" if ok else "FAIL")
