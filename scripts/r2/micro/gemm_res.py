"""bf16 C += A B (the dX form with the gradient residual) at the c4 shapes: wide (global residual) vs KL_GEMM_NOWIDE_R."""
import os, sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
_capi.lib()
def t(fn, n=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
for name, K in (("qkv dX", 1536), ("hsp dS", 640), ("out dX", 512)):
    A = (torch.randn(32, 4096, K, device="cuda") / 22).bfloat16()
    W = (torch.randn(K, 512, device="cuda") / 22).bfloat16()
    C = torch.randn(32, 4096, 512, device="cuda").bfloat16()
    ms = t(lambda: _capi.gemm(A, W, C, beta=1.0))
    print(f"{name} {os.environ.get('KL_GEMM_NOWIDE_R') and 'nowide' or 'wide'}: {ms*1e3:.1f} us", flush=True)
