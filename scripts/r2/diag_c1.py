import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2602_10016_b200.configs import CONFIGS
from paper_2602_10016_b200.model import KunlunModel
from paper_2602_10016_b200.optim import FlatAdam, TrainStep
from paper_2602_10016_b200.synth import ctr_batch
from paper_2602_10016_b200.tensor import raise_if_nonfinite, NumericsError
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
cfg, B = CONFIGS[name]()
dev = torch.device("cuda", 0)
model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
opt = FlatAdam(model.P)
Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=1234)
X = torch.tensor(Xn, device=dev).bfloat16(); S = [torch.tensor(s, device=dev).bfloat16() for s in Sn]
lens = [torch.tensor(l, device=dev) for l in Ln]; y = torch.tensor(yn, device=dev)
st = TrainStep(model, opt, X, S, lens, y, None)
for i in range(30):
    loss = st.eager()
    torch.cuda.synchronize()
    g = model.P.gflat
    p = model.P.flat
    print(i, float(loss), "grad finite", bool(torch.isfinite(g).all()), "param finite", bool(torch.isfinite(p).all()),
          "gmax", float(g.abs().max()))
    try:
        raise_if_nonfinite(dev)
    except NumericsError as e:
        print("  NumericsError at step", i)
        bad = [n for n in model.P.names() if not torch.isfinite(model.P.grad(n)).all()]
        print("  nonfinite grads:", bad[:10])
        break
