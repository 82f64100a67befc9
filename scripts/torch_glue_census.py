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

with profile(activities=[ProfilerActivity.CPU], with_stack=True) as prof:
    st.eager()
    torch.cuda.synchronize()
agg = collections.Counter()
for ev in prof.events():
    name = ev.name
    if not name.startswith("aten::") or name in ("aten::empty", "aten::empty_strided", "aten::view", "aten::as_strided",
                                                  "aten::reshape", "aten::slice", "aten::select", "aten::t",
                                                  "aten::transpose", "aten::permute", "aten::expand", "aten::detach",
                                                  "aten::unsqueeze", "aten::squeeze", "aten::alias", "aten::lift_fresh",
                                                  "aten::_reshape_alias", "aten::resize_", "aten::set_",
                                                  "aten::result_type", "aten::is_nonzero", "aten::item",
                                                  "aten::_local_scalar_dense", "aten::empty_like", "aten::split",
                                                  "aten::narrow", "aten::unbind", "aten::chunk", "aten::_unsafe_view"):
        continue
    frames = [f for f in (ev.stack or []) if "paper_2602_10016_b200" in f]
    site = frames[0].split("paper_2602_10016_b200/")[-1] if frames else "(autograd engine)"
    agg[(name, site)] += 1
for (name, site), c in agg.most_common(60):
    print(f"{c:4d}  {name:28s} {site}")
