"""Standalone probe of the tcgen05 SWA kernels (run under `timeout` on the GPU
box): fwd, then bwd, on one small bf16 case, compared with the SIMT kernels."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi  # noqa: E402
from paper_2602_10016_b200 import functional as F  # noqa: E402

stage = sys.argv[1]
B, T, H, dh, w = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), 64, int(sys.argv[5])
causal = len(sys.argv) > 6 and sys.argv[6] == "1"
lens_arg = None
if len(sys.argv) > 7:
    lens_arg = [T] * B if sys.argv[7] == "full" else [int(x) for x in sys.argv[7].split(",")]
    assert len(lens_arg) == B, "need one length per sample"
g = torch.Generator(device="cuda").manual_seed(0)
qkv = torch.randn(B, T, 3 * H * dh, device="cuda", generator=g).to(torch.bfloat16)
lens = torch.tensor(lens_arg or [T - 3 * i for i in range(B)], device="cuda", dtype=torch.int32).clamp_min(0)
L = _capi.lib()
outs = {}
for path in ((0,) if stage.endswith("only") else (1, 0)):  # SIMT, then auto (tcgen05)
    L.kl_set_gemm_path(path)
    q = qkv.clone().requires_grad_(True)
    o = F.swa_core(q, lens, H, dh, w, causal)
    torch.cuda.synchronize()
    print("fwd done path", path, flush=True)
    if stage.startswith("bwd"):
        go = torch.randn(o.shape, device="cuda", generator=torch.Generator(device="cuda").manual_seed(1)).to(o.dtype)
        o.backward(go)
        torch.cuda.synchronize()
        print("bwd done path", path, flush=True)
        outs[path] = (o.detach().float(), q.grad.float())
    else:
        outs[path] = (o.detach().float(), None)
if len(outs) < 2:
    sys.exit(0)
a, b = outs[1], outs[0]
print("fwd max|diff|", float((a[0] - b[0]).abs().max()), "max|ref|", float(b[0].abs().max()))
if stage.startswith("bwd"):
    print("bwd max|diff|", float((a[1] - b[1]).abs().max()), "max|ref|", float(b[1].abs().max()))
