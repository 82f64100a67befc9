"""A/B the tcgen05 (operand-swapped) and SIMT paths on the model's batched
small products (graph-replayed per-call device time):  python scripts/probes/gemm_small_ab.py"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi  # noqa: E402
from paper_2602_10016_b200._capi import gemm  # noqa: E402

bf = torch.bfloat16
dev = "cuda"
B, H = 128, 4
k = torch.randn(B, H, 16, 64, device=dev).to(bf)
wq = torch.randn(H, 64, 256, device=dev).to(bf)
pool = torch.randn(4, 16, device=dev).to(bf)
X = torch.randn(B, 16, 256, device=dev).to(bf)
agg = torch.randn(16, 48, device=dev).to(bf)
st = torch.randn(B, 48, 256, device=dev).to(bf)
g16 = torch.randn(B, H, 16, 256, device=dev).to(bf)
wg = torch.zeros(H, 64, 256, device=dev)
cases = {
    "fold_kv 16x256x64 b128x4": lambda: gemm(k, wq),
    "pool 4x256x16 b128": lambda: gemm(pool, X),
    "agg 16x256x48 b128 (+res)": lambda: gemm(agg, st, residual=X),
    "fold bwd dK 16x64x256 b128x4": lambda: gemm(g16, wq.transpose(1, 2)),
    "fold bwd dW 64x256x16 red b": lambda: gemm(k.transpose(2, 3), g16, wg.unsqueeze(0), beta=1.0, reduce=(True, False)),
}


def timeit(fn, n=30):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
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
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


for name, fn in cases.items():
    res = []
    for label, path, swap in (("tc+swap", 0, True), ("tc", 0, False), ("simt", 1, False)):
        _capi.SWAP_SMALL_M = swap
        _capi.lib().kl_set_gemm_path(path)
        try:
            res.append(f"{label} {timeit(fn):6.1f}us")
        except Exception as exc:  # noqa: BLE001
            res.append(f"{label} n/a ({str(exc)[:40]})")
    _capi.SWAP_SMALL_M = False
    _capi.lib().kl_set_gemm_path(0)
    print(f"{name:32s} " + "  ".join(res))
