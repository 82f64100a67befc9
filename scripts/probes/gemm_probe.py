"""GEMM timing probe on the B200: kl_gemm on model shapes, CUDA-event timed.
usage: python scripts/probes/gemm_probe.py [reps]"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200._capi import gemm  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g = torch.Generator(device="cuda").manual_seed(0)
bf = torch.bfloat16


def t(fn):
    fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


B, T, d = 128, 1024, 256
S = torch.randn(B, T, d, device="cuda", generator=g).to(bf)
Wqkv = torch.randn(3 * d, d, device="cuda", generator=g).to(bf)
Wo = torch.randn(d, d, device="cuda", generator=g).to(bf)
O = torch.randn(B, T, d, device="cuda", generator=g).to(bf)
qkv = torch.empty(B, T, 3 * d, device="cuda", dtype=bf)
out = torch.empty(B, T, d, device="cuda", dtype=bf)
dW = torch.zeros(3 * d, d, device="cuda")
cases = {
    "qkv_fwd  (131072x768x256)": lambda: gemm(S, Wqkv.t(), qkv),
    "oproj+res(131072x256x256)": lambda: gemm(O, Wo.t(), out, residual=S),
    "oproj    (131072x256x256)": lambda: gemm(O, Wo.t(), out),
    "dgrad qkv(131072x256x768)": lambda: gemm(qkv, Wqkv, out),
    "wgrad qkv(768x256xK=131072)": lambda: gemm(qkv.transpose(1, 2).unsqueeze(0), S.unsqueeze(0), dW.view(1, 1, 768, 256),
                                                beta=1.0, reduce=(True, True)),
}
for name, fn in cases.items():
    ms = t(fn)
    M, N, K = {"qkv_fwd": (131072, 768, 256), "oproj+res": (131072, 256, 256), "oproj   ": (131072, 256, 256),
               "dgrad qkv": (131072, 256, 768), "wgrad qkv": (768, 256, 131072)}[name[:9].rstrip() if name[:9].rstrip() in ("qkv_fwd", "oproj+res", "dgrad qkv", "wgrad qkv") else "oproj   "]
    print(f"{name}: {ms * 1e3:8.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s", flush=True)

bias = torch.randn(d, device="cuda", generator=g)
out32 = torch.empty(B, T, d, device="cuda")
S32 = torch.randn(B, T, d, device="cuda", generator=g)
more = {
    "beta=1 (C read)": lambda: gemm(O, Wo.t(), out, beta=1.0),
    "bias": lambda: gemm(O, Wo.t(), out, bias=bias),
    "act silu": lambda: gemm(O, Wo.t(), out, acts=["silu"]),
    "res fp32 out": lambda: gemm(O, Wo.t(), out32, residual=S32),
    "res = out (inplace)": lambda: gemm(O, Wo.t(), out, residual=out),
}
for name, fn in more.items():
    print(f"{name}: {t(fn) * 1e3:8.1f} us", flush=True)
