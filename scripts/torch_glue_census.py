"""Profile one eager training step (c2) and list the torch-native (non-kl)
kernels with the Python call site in this package that issued them."""
import collections
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2602_10016_b200.configs import CONFIGS  # noqa: E402
from paper_2602_10016_b200.model import KunlunModel  # noqa: E402
from paper_2602_10016_b200.optim import FlatAdam, TrainStep  # noqa: E402
from paper_2602_10016_b200.synth import ctr_batch  # noqa: E402

cfg, B = CONFIGS["c2"]()
dev = torch.device("cuda", 0)
model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
opt = FlatAdam(model.P)
Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=1)
X = torch.tensor(Xn, device=dev).bfloat16()
S = [torch.tensor(s, device=dev).bfloat16() for s in Sn]
L = [torch.tensor(l, device=dev) for l in Ln]
y = torch.tensor(yn, device=dev)
st = TrainStep(model, opt, X, S, L, y)
for _ in range(3):
    st.eager()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CPU], with_stack=True, record_shapes=True) as prof:
    st.eager()
    torch.cuda.synchronize()
agg = collections.Counter()
KEEP = ("aten::copy_", "aten::add_", "aten::fill_", "aten::cat", "aten::zero_", "aten::mul", "aten::sum",
        "aten::linalg_vecdot", "aten::add", "aten::clone", "aten::_to_copy", "aten::ones_like", "aten::stack")
for ev in prof.events():
    if ev.name not in KEEP:
        continue
    # skip nested (e.g. copy_ inside clone): keep only events without a KEEP parent
    par = ev.cpu_parent
    nested = False
    while par is not None:
        if par.name in KEEP:
            nested = True
            break
        par = par.cpu_parent
    if nested:
        continue
    shapes = str(ev.input_shapes)[:90]
    stack = [f for f in (ev.stack or []) if "paper_2602_10016_b200" in f or "/tests/" in f]
    site = stack[0].split("/")[-1] if stack else ""
    agg[(ev.name, shapes, site)] += 1
for (name, shapes, site), c in agg.most_common(45):
    print(f"{c:4d}  {name:22s} {shapes:92s} {site}")
