import sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
from paper_2602_10016_b200._capi import gemm
_capi.lib()
g = torch.Generator(device="cuda").manual_seed(11)
def rel(a, b):
    return float((a.double() - b.double()).abs().max() / b.double().abs().max())
for (M, N, K) in ((32768, 512, 1536), (37000, 1024, 1600), (65536, 512, 2048)):
    for bmn in (False, True):
        A = (torch.randn(M, K, device="cuda", generator=g) * 0.05).bfloat16()
        Bt = (torch.randn(N, K, device="cuda", generator=g) * 0.05).bfloat16()
        B = Bt.t().contiguous() if bmn else Bt.t()
        ref = A.double() @ B.double()
        _capi.reset_path_hits()
        out = gemm(A, B)
        w = _capi.path_hits()["gemm_wide"]
        out32 = gemm(A, B, out_dtype=torch.float32)
        bias = torch.randn(N, device="cuda", generator=g)
        ob = gemm(A, B, bias=bias)
        print(M, N, K, "B MN" if bmn else "B K", "wide", w, "plain bf16", f"{rel(out, ref):.2e}", "fp32", f"{rel(out32, ref):.2e}",
              "bias", f"{rel(ob, ref + bias.double()):.2e}", "nan", int(torch.isnan(out).sum()), flush=True)
