"""Per-call device time of small kl_gemm shapes, back to back (eager) and
replayed from a CUDA graph:  python scripts/probes/gemm_latency.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi  # noqa: E402
from paper_2602_10016_b200._capi import gemm  # noqa: E402

bf = torch.bfloat16
dev = "cuda"
x = torch.randn(128, 32, 256, device=dev).to(bf)
w = torch.randn(256, 256, device=dev).to(bf)
big = torch.randn(3072, 256, device=dev).to(bf)
w2 = torch.randn(512, 256, device=dev).to(bf)
o32 = torch.zeros(256, 256, device=dev)
q32 = torch.randn(32, 4, 64, device=dev)
wk = torch.randn(4, 64, 256, device=dev)
xs = torch.randn(32, 256, device=dev)
wq = torch.randn(256, 256, device=dev)
cases = {
    "fp32 32x256x256": lambda: gemm(xs, wq.t()),
    "fp32 32x256x64 b4": lambda: gemm(q32.permute(1, 0, 2), wk),
    "fp32 dW 256x256 K=32 +=": lambda: gemm(wq[:, :32], xs, o32, beta=1.0),
    "torch add (tiny)": lambda: torch.add(o32, 1.0),
    "4096x256x256 plain": lambda: gemm(x.view(-1, 256), w.t()),
    "3072x512x256 plain": lambda: gemm(big, w2.t()),
    "3072x512x256 bias+silu+aux": lambda: gemm(big, w2.t(), bias=torch.zeros(512, device=dev), acts=["silu"],
                                               aux=torch.empty(3072, 512, device=dev, dtype=bf), aux_mode=1),
    "dW 256x256 K=4096 fp32+=": lambda: gemm(x.view(-1, 256).t(), x.view(-1, 256), o32, beta=1.0),
    "b128 32x256x256": lambda: gemm(x, w.t()),
}
for name, fn in cases.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    n = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / n * 1e3
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n):
                fn()
    torch.cuda.synchronize()
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    graph = e0.elapsed_time(e1) / n * 1e3
    print(f"{name:32s} eager {eager:7.1f} us/call   graph {graph:7.1f} us/call   path {_capi.lib().kl_last_gemm_path()}")
