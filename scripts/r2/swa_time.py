"""Isolated timing of the tcgen05 SWA kernels at the bench shapes (CUDA
events over 50 reps, after warm-up): fwd (swa_fwd_tc3) and bwd (rowdot +
dkv + dq) for c4 (B=32, H=8, T=4096) and c2 (B=128, H=4, T=1024)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
from paper_2602_10016_b200 import functional as F

_capi.lib()
for name, B, H, T in (("c4", 32, 8, 4096), ("c2", 128, 4, 1024)):
    torch.manual_seed(0)
    qkv = (torch.randn(B, T, 3 * H * 64, device="cuda") * 0.5).bfloat16().requires_grad_(True)
    lens = torch.randint(T // 2, T + 1, (B,), device="cuda", dtype=torch.int32)
    lens[0] = T
    o = F.swa_core(qkv, lens, H, 64, 128, False)
    g = torch.randn_like(o)
    o.backward(g)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    reps = 50
    ev[0].record()
    for _ in range(reps):
        o = F.swa_core(qkv, lens, H, 64, 128, False)
    ev[1].record()
    for _ in range(reps):
        qkv.grad = None
        o.backward(g, retain_graph=True)
    ev[2].record()
    torch.cuda.synchronize()
    print(f"{name}: swa fwd {ev[0].elapsed_time(ev[1]) / reps * 1e3:7.1f} us   bwd {ev[1].elapsed_time(ev[2]) / reps * 1e3:7.1f} us")
