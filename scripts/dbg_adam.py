import sys, numpy as np, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import functional as F
from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig
from paper_2602_10016_b200.optim import FlatAdam, TrainStep
from paper_2602_10016_b200.synth import ctr_batch
cfg = ModelConfig(L=3, d=256, heads=4, n_ctx=16, compskip=True, events=[EventConfig(T=256, w=64, budget=32, n_seeds=32, rank=8)])
dev = torch.device("cuda", 0)
Xn, Sn, Ln, yn = ctr_batch(cfg, 8, seed=5)
res = []
for split in (False, True):
    F.BRANCH_STREAMS = split
    model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
    batch = (torch.tensor(Xn, device=dev).bfloat16(), [torch.tensor(s, device=dev).bfloat16() for s in Sn], [torch.tensor(l, device=dev) for l in Ln], torch.tensor(yn, device=dev))
    opt = FlatAdam(model.P, lr=1e-3)
    st = TrainStep(model, opt, *batch[:3], batch[3])
    for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
        st.eager()
    torch.cuda.synchronize()
    res.append((model, model.P.flat.detach().clone(), model.P.gflat.detach().clone(), opt.m.clone(), int(opt.t.item())))
    if split:
        print('segments', st.segments, 'late', st.late)
m0, f0, g0, mm0, t0 = res[0]; m1, f1, g1, mm1, t1 = res[1]
print('t', t0, t1, 'grad maxdiff', float((g1 - g0).abs().max()), 'm maxdiff', float((mm1 - mm0).abs().max()))
P = m0.P
for key, (off, shape) in P._blocks.items():
    n = int(np.prod(shape)) if shape else 1
    d = float((f1[off:off+n] - f0[off:off+n]).abs().max())
    if d > 1e-6:
        print('block', key, shape, off, 'param diff', d, 'grad diff', float((g1[off:off+n]-g0[off:off+n]).abs().max()), 'm diff', float((mm1[off:off+n]-mm0[off:off+n]).abs().max()))
