import sys, torch, numpy as np, traceback
sys.path.insert(0, ".")
from paper_2602_10016_b200.configs import CONFIGS
from paper_2602_10016_b200.model import KunlunModel
from paper_2602_10016_b200.synth import ctr_batch
from paper_2602_10016_b200 import functional as F
from paper_2602_10016_b200.tensor import set_numerics_check
cfg, B = CONFIGS["c1"]()
dev = torch.device("cuda", 0)
Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=1234)
print("lengths", [l[:12] for l in Ln], Xn.shape, [s.shape for s in Sn], "X finite", np.isfinite(Xn).all(), [np.isfinite(s).all() for s in Sn])
for tog in [{}, {"GDPA_FUSED": False}, {"HSP_FUSED": False}, {"BRANCH_STREAMS": False}]:
    for k, v in tog.items(): setattr(F, k, v)
    model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
    X = torch.tensor(Xn, device=dev).bfloat16(); S = [torch.tensor(s, device=dev).bfloat16() for s in Sn]
    lens = [torch.tensor(l, device=dev) for l in Ln]
    set_numerics_check("eager")
    try:
        with torch.no_grad():
            lg = model.forward(X, S, lens)
        print(tog, "ok", float(lg.abs().max()))
    except Exception as e:
        print(tog, "ERR", e)
        traceback.print_exc(limit=-6)
    set_numerics_check("deferred")
    for k, v in tog.items(): setattr(F, k, True)
