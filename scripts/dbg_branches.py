import sys, numpy as np, torch
sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from test_gpu_branches import _run
from paper_2602_10016_b200 import functional as F
from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig
from paper_2602_10016_b200.synth import ctr_batch
cfg = ModelConfig(L=3, d=256, heads=4, n_ctx=16, compskip=False, events=[EventConfig(T=384, w=128, budget=32, n_seeds=32, rank=8)])
dev = torch.device("cuda", 0)
model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
Xn, Sn, Ln, yn = ctr_batch(cfg, 8, seed=3)
Ln = [np.array([384, 200, 1, 0, 384, 383, 129, 64], dtype=np.int32)]
batch = (torch.tensor(Xn, device=dev).bfloat16(), [torch.tensor(s, device=dev).bfloat16() for s in Sn], [torch.tensor(l, device=dev) for l in Ln], torch.tensor(yn, device=dev))
res = {}
for bs in (False, True):
    F.BRANCH_STREAMS = bs
    for graph in (False, True, False):
        l, _, g = _run(model, batch, graph)
        res.setdefault((bs, graph), []).append((l, g))
l0, g0 = res[(False, False)][0]
sc = float(g0.abs().max())
names = model.P.names()
for k, v in res.items():
    for l, g in v:
        d = (g - g0).abs()
        i = int(d.argmax())
        # find param containing index i
        owner = None
        for n in names:
            blk = model.P.block_of(n) if hasattr(model.P, 'block_of') else None
        print(k, 'loss', l, 'dl', l - l0, 'max rel', float(d.max()) / sc, 'argmax', i)
# locate the worst block for graph+streams
l2, g2 = res[(True, True)][0]
d = (g2 - g0).abs()
for key, (off, shape) in model.P._blocks.items():
    n = int(np.prod(shape)) if shape else 1
    m = float(d[off:off + n].max()) if n else 0
    if m > 1e-3 * sc:
        print('block', key, shape, 'maxdiff/scale', m / sc, 'blockmax/scale', float(g0[off:off+n].abs().max()) / sc)
