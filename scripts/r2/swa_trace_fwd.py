"""Pipeline clock stamps of CTA 0 of the tcgen05 SWA forward (KL_SWA_TRACE_FWD; lib built with -DKL_SWA_TRACE_BUILD)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
from paper_2602_10016_b200 import functional as F
_capi.lib()
B, H, T = 32, 8, 4096
torch.manual_seed(0)
qkv = (torch.randn(B, T, 3 * H * 64, device="cuda") * 0.5).bfloat16()
lens = torch.full((B,), T, device="cuda", dtype=torch.int32)
o = F.swa_core(qkv, lens, H, 64, 128, False)
tr = torch.zeros(20 * 1024, dtype=torch.int64, device="cuda")
os.environ["KL_SWA_TRACE_FWD"] = str(tr.data_ptr())
torch.cuda.synchronize()
o = F.swa_core(qkv, lens, H, 64, 128, False)
torch.cuda.synchronize()
del os.environ["KL_SWA_TRACE_FWD"]
t = tr.view(20, 1024).cpu().numpy().astype(np.int64)
base = t[t > 0].min()
t = np.where(t > 0, t - base, -1)
n_items = int((t[6] >= 0).sum())
print("items", n_items, "tiles", int((t[10] >= 0).sum()))
print("item:  w1start  w1kvok  w1issue | smwait  smgotS  sm_pwait sm_pok smdone | w2wait w2issue")
for n in list(range(0, 30)) + list(range(150, 160)):
    print(f"{n:4d}: " + " ".join(f"{t[e][n]:8d}" for e in (0, 1, 2, 5, 6, 7, 8, 9, 3, 4)))
print("tiles: tma | o wait, got, end")
for k in range(0, 10):
    print(k, t[10][k], "|", t[11][k], t[12][k], t[13][k])
v = lambda e: t[e][:n_items]
d = lambda a, b: np.median((v(b) - v(a))[10:n_items - 10])
print("median period (w1 issue)", np.median(np.diff(v(2)[10:n_items - 10])))
print("sm: wait S", d(5, 6), " S->max done", d(6, 7), " p_empty wait", d(7, 8), " exp+store", d(8, 9), " done->w2 issue", d(9, 4))
print("w1: kv wait", d(0, 1), " s_empty wait", d(1, 2))
