"""Standalone timing probe of the fused GDPA kernels (kl_gdpa_fwd/bwd) at a
given shape (run on the GPU box; also the ncu target):
    python scripts/probes/gdpa_probe.py [B T d] [iters]
Prints average device time per launch and the achieved algorithmic HBM
bandwidth (fwd: read S + write Y; bwd: read S, dY + write dS)."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi  # noqa: E402
from paper_2602_10016_b200 import functional as F  # noqa: E402

B, T, d = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (128, 1024, 256)
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20
HK, n_kv = 64, 16
torch.manual_seed(0)
S = (torch.randn(B, T, d, device="cuda") / d ** 0.5).bfloat16()
Kt = (torch.randn(B, HK, d, device="cuda") / 2).bfloat16()
Vt = (torch.randn(B, HK, d, device="cuda") / 8).bfloat16()
G = torch.randn(B, T, d, device="cuda").bfloat16()
lengths = torch.randint(T // 2, T + 1, (B,), device="cuda", dtype=torch.int32)
Y, dS = torch.empty_like(S), torch.empty_like(S)
dKt, dVt = torch.empty_like(Kt), torch.empty_like(Vt)
codes = F._codes(("silu", "relu", "identity", "tanh"))
a = F._gdpa_args(S, Kt, Vt, lengths, codes, n_kv, 1.0 / T)
a.Y, a.dY, a.dS, a.dKt, a.dVt = Y.data_ptr(), G.data_ptr(), dS.data_ptr(), dKt.data_ptr(), dVt.data_ptr()
st = torch.cuda.current_stream().cuda_stream
L = _capi.lib()


def run(name):
    for _ in range(3):
        _capi._check(getattr(L, name)(C.byref(a), st), name)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        getattr(L, name)(C.byref(a), st)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters


which = sys.argv[5] if len(sys.argv) > 5 else "both"
row = B * T * d * 2
if which in ("both", "fwd"):
    ms = run("kl_gdpa_fwd")
    print(f"gdpa_fwd  B={B} T={T} d={d}: {ms * 1e3:8.1f} us  {2 * row / ms / 1e6:7.0f} GB/s")
if which in ("both", "bwd"):
    ms = run("kl_gdpa_bwd")
    print(f"gdpa_bwd  B={B} T={T} d={d}: {ms * 1e3:8.1f} us  {3 * row / ms / 1e6:7.0f} GB/s")

if len(sys.argv) > 6 and sys.argv[6] == "trace":
    tr = torch.zeros(32 * 16, dtype=torch.int64, device="cuda")
    a.trace = tr.data_ptr()
    for name in ("kl_gdpa_fwd", "kl_gdpa_bwd"):
        tr.zero_()
        getattr(L, name)(C.byref(a), st)
        torch.cuda.synchronize()
        t = tr.view(32, 16).cpu()
        t0 = int(t[0][t[0] > 0].min()) if (t[0] > 0).any() else 0
        print(name, "stage clocks (relative to first stamp), rows = tiles of CTA 0")
        for c in range(32):
            if (t[c] > 0).any():
                print(c, " ".join(f"{int(v) - t0:7d}" if v > 0 else "      ." for v in t[c][:11]))
