"""Attribute the eager ATen kernels of one training step to Python source
lines (torch.profiler with stacks): which copies / cats / fills / adds the
step launches besides the C-ABI kernels."""
import collections
import sys

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi, configs
from paper_2602_10016_b200.model import KunlunModel
from paper_2602_10016_b200.optim import FlatAdam, TrainStep
from paper_2602_10016_b200.synth import ctr_batch
from paper_2602_10016_b200.grouped import stage

name = sys.argv[1] if len(sys.argv) > 1 else "c4"
cfg, B = configs.CONFIGS[name]()
_capi.lib()
m = KunlunModel(cfg, "cuda", torch.bfloat16)
Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=1)
X = torch.tensor(Xn, device="cuda").bfloat16()
S = [torch.tensor(s, device="cuda").bfloat16() for s in Sn]
L = [torch.tensor(l, device="cuda") for l in Ln]
if m.groups is not None:
    S, L = stage(S), stage(L)
y = torch.tensor(yn, device="cuda")
st = TrainStep(m, FlatAdam(m.P), X, S, L, y)
for _ in range(2):
    st.eager()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA], with_stack=True, record_shapes=True) as prof:
    st.eager()
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if not e.name.startswith("aten::") or e.name in ("aten::empty", "aten::view", "aten::as_strided",
                                                      "aten::empty_strided", "aten::slice", "aten::select",
                                                      "aten::transpose", "aten::permute", "aten::unsqueeze",
                                                      "aten::expand", "aten::reshape", "aten::t", "aten::alias",
                                                      "aten::_reshape_alias", "aten::unbind", "aten::squeeze",
                                                      "aten::detach", "aten::lift_fresh", "aten::result_type",
                                                      "aten::resolve_conj", "aten::resolve_neg", "aten::record_stream",
                                                      "aten::is_nonzero", "aten::item", "aten::_local_scalar_dense",
                                                      "aten::empty_like", "aten::split", "aten::narrow", "aten::chunk"):
        continue
    dev_us = getattr(e, "device_time_total", 0) or getattr(e, "cuda_time_total", 0)
    if dev_us <= 0:
        continue
    frames = [f for f in (e.stack or []) if "paper_2602" in f or "bench" in f]
    src = frames[0] if frames else ("bwd" if not e.stack else "?" + str(e.stack[:2]))
    key = (e.name, src, str(e.input_shapes)[:90] if src == "bwd" else "")
    agg[key][0] += 1
    agg[key][1] += dev_us
tot = sum(v[1] for v in agg.values())
print(f"ATen device time {tot:.0f} us in {sum(v[0] for v in agg.values())} ops")
for (n, src, sh), (c, us) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:60]:
    print(f"{us:8.0f} us {c:4d}x {n:24s} {src} {sh}")
