import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2602_10016_b200 import attention as A, functional as F, _capi
from paper_2602_10016_b200.tensor import Params
for B in (5, 8, 16, 32):
    rng = np.random.default_rng(0)
    P = Params(); mp = A.MhaParams.create(P, "m", 64, 4, rng); P.finalize("cuda", torch.bfloat16)
    s = torch.tensor(rng.normal(0, 0.125, (B, 256, 64)), device="cuda").bfloat16()
    lens = torch.full((B,), 256, dtype=torch.int32, device="cuda")
    qkv = F.linear(s, P, mp.wqkv)
    o = F.swa_core(qkv, lens, 4, 16, 64, False)
    y = F.linear(o, P, mp.wout, residual=s)
    torch.cuda.synchronize()
    f = lambda t: bool(torch.isfinite(t.float()).all())
    bad_o = (~torch.isfinite(o.float())).nonzero()
    print(B, "qkv", f(qkv), "o", f(o), "y", f(y), "first bad o", bad_o[:3].tolist(), "n bad", bad_o.shape[0])
