"""Probe of the fused HSP pooling kernels vs a torch fp32 reference:
    python scripts/probes/hsp_probe.py [B T d HQ n1]"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi  # noqa: E402

B, T, d, HQ, n1 = (int(x) for x in (sys.argv[1:6] if len(sys.argv) > 5 else (8, 1024, 256, 160, 128)))
g = torch.Generator(device="cuda").manual_seed(0)
S = (torch.randn(B, T, d, device="cuda", generator=g) / d ** 0.5).to(torch.bfloat16)
Q = (torch.randn(HQ, d, device="cuda", generator=g) * 2.0).to(torch.bfloat16)
lens = torch.randint(0, T + 1, (B,), device="cuda", generator=g).to(torch.int32)
lens[0] = T
if B > 1:
    lens[1] = 0
if B > 2:
    lens[2] = 1
import os  # noqa: E402

if os.environ.get("LENS"):
    lens = torch.tensor([int(x) for x in os.environ["LENS"].split(",")], device="cuda", dtype=torch.int32)
O1 = torch.full((B, n1, d), 7.0, device="cuda", dtype=torch.bfloat16)
O2 = torch.full((B, max(HQ - n1, 1), d), 7.0, device="cuda", dtype=torch.bfloat16)
LSE = torch.zeros(B, HQ, device="cuda")
a = _capi.HspArgs()
a.B, a.T, a.HQ, a.d, a.n1, a.dtype = B, T, HQ, d, n1, _capi.KL_BF16
a.lengths = lens.data_ptr()
a.S, a.s_rs, a.s_bs = S.data_ptr(), S.stride(1), S.stride(0)
a.Q = Q.data_ptr()
a.O1, a.o1_bs, a.O2, a.o2_bs = O1.data_ptr(), O1.stride(0), O2.data_ptr(), O2.stride(0)
a.LSE = LSE.data_ptr()
if os.environ.get("TRACE"):
    import time

    tr = torch.zeros(148 * 8 * 4, dtype=torch.int32).pin_memory()
    os.environ["KL_HSP_TRACE"] = str(tr.data_ptr())
    _capi.call("kl_hsp_fwd", C.byref(a), _capi._stream())
    time.sleep(3)
    t = tr.view(148, 8, 4)
    for cta in range(int(os.environ.get("TRACE"))):
        print("cta", cta, [tuple(t[cta, r].tolist()) for r in range(6)], flush=True)
    os._exit(3)
_capi.call("kl_hsp_fwd", C.byref(a), _capi._stream())
torch.cuda.synchronize()
# reference
Z = torch.einsum("qd,btd->bqt", Q.float(), S.float())
mask = torch.arange(T, device="cuda")[None, None, :] < lens[:, None, None]
Zm = Z.masked_fill(~mask, float("-inf"))
lse = torch.logsumexp(Zm, dim=-1)
P = torch.softmax(Zm, dim=-1).nan_to_num(0.0)
O = torch.einsum("bqt,btd->bqd", P, S.float())
out = torch.cat([O1.float(), O2.float()[:, : HQ - n1]], dim=1)
err = (out - O).abs().max().item() / O.abs().max().item()
ok = lens > 0
lerr = (LSE[ok] - lse[ok]).abs().max().item()
print(f"fwd: pooled rel err {err:.3e}, lse abs err {lerr:.3e}, empty rows zero {bool((out[~ok] == 0).all())}, "
      f"lse inf {bool(torch.isinf(LSE[~ok]).all())}")
n = 20
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n):
    _capi.call("kl_hsp_fwd", C.byref(a), _capi._stream())
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
fl = 4.0 * B * HQ * T * d
print(f"fwd time {ms * 1e3:.1f} us, {fl / ms / 1e9:.1f} TF/s (algorithmic, full T)")
