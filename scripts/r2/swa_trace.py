"""Pipeline clock stamps of CTA 0 of the tcgen05 dK/dV kernel (KL_SWA_TRACE) at the c4 shape."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
from paper_2602_10016_b200 import functional as F
_capi.lib()
B, H, T = 32, 8, 4096
torch.manual_seed(0)
qkv = (torch.randn(B, T, 3 * H * 64, device="cuda") * 0.5).bfloat16().requires_grad_(True)
lens = torch.full((B,), T, device="cuda", dtype=torch.int32)
o = F.swa_core(qkv, lens, H, 64, 128, False)
g = torch.randn_like(o)
o.backward(g, retain_graph=True)
tr = torch.zeros(20 * 1024, dtype=torch.int64, device="cuda")
os.environ["KL_SWA_TRACE"] = str(tr.data_ptr())
torch.cuda.synchronize()
qkv.grad = None
o.backward(g, retain_graph=True)
torch.cuda.synchronize()
del os.environ["KL_SWA_TRACE"]
t = tr.view(20, 1024).cpu().numpy().astype(np.int64)
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
names = {0: "w1 loop", 1: "w1 kv/qg ok", 2: "w1 sd_empty ok (issue S)", 3: "w10 loop", 4: "w10 pd_full ok (issue dV/dK)",
         5: "wg wait S", 6: "wg got S", 7: "wg done", 8: "epi wait acc", 9: "epi got acc", 10: "tma tile"}
n_items = int((t[6] >= 0).sum())
print("items traced", n_items, "tiles", int((t[10] >= 0).sum()))
print("item:  w1start  w1kvok  w1issue | wgwait  wggotS  wgdone | w10wait w10issue")
for n in list(range(0, 40)) + list(range(200, 215)):
    print(f"{n:4d}: " + " ".join(f"{t[e][n]:8d}" for e in (0, 1, 2, 5, 6, 7, 3, 4)))
print("tiles: tma | epi wait, got, end | wg0: top, staged, bar, items | wg1: top, staged, bar, items")
for k in range(0, 14):
    print(k, t[10][k], "|", t[8][k], t[9][k], t[19][k], "|", t[11][k], t[13][k], t[15][k], t[17][k], "|", t[12][k], t[14][k], t[16][k], t[18][k])
v = lambda e: t[e][:n_items]
d = lambda a, b: np.median((v(b) - v(a))[10:n_items - 10])
print("median per-item period (w1 issue)", np.median(np.diff(v(2)[10:n_items - 10])))
print("median wg S wait (got-wait)", d(5, 6), "wg math (done-got)", d(6, 7), "S ready->w10 issue", d(7, 4))
print("median w1: loop->kvok", d(0, 1), " kvok->sd_empty ok", d(1, 2))
print("median w10: wait->pd ok", d(3, 4))
