"""Time model-shaped kl_gemm calls (CUDA events, L2-resident or not):
    python scripts/probes/gemm_bench.py  -> one line per shape: us, TF/s, GB/s."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200._capi import gemm  # noqa: E402

bf = torch.bfloat16
g = torch.Generator(device="cuda").manual_seed(0)
B, T, d = 128, 1024, 256
S = torch.randn(B, T, d, device="cuda", generator=g).to(bf)
W3 = torch.randn(3 * d, d, device="cuda", generator=g).to(bf)
bias = torch.randn(3 * d, device="cuda", generator=g)
out3 = torch.empty(B, T, 3 * d, device="cuda", dtype=bf)
out1 = torch.empty(B, T, d, device="cuda", dtype=bf)
dW = torch.zeros(3 * d, d, device="cuda")
G3 = torch.randn(B, T, 3 * d, device="cuda", generator=g).to(bf)
cases = {
    "qkv  (128K x 768 x 256)": (lambda: gemm(S, W3.t(), out3), 2 * B * T * 768 * 256, B * T * (256 + 768) * 2),
    "bias+relu (128K x 256 x 256)": (lambda: gemm(S, W3[:d].t(), out1, bias=bias[:d], acts=["relu"]),
                                     2 * B * T * 256 * 256, B * T * 512 * 2),
    "residual (128K x 256 x 256)": (lambda: gemm(S, W3[:d].t(), out1, residual=S), 2 * B * T * 256 * 256,
                                    B * T * 768 * 2),
    "dX  (128K x 256 x 768)": (lambda: gemm(G3, W3, out1), 2 * B * T * 768 * 256, B * T * (768 + 256) * 2),
    "dW  (768 x 256, K=128K, fp32 +=)": (lambda: gemm(G3.view(-1, 768).t(), S.view(-1, 256), dW, beta=1.0),
                                        2 * B * T * 768 * 256, B * T * (768 + 256) * 2),
}
for name, (fn, flops, byts) in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 20
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    print(f"{name:36s} {ms * 1e3:8.1f} us  {flops / ms / 1e9:7.1f} TF/s  {byts / ms / 1e6:7.0f} GB/s")
