"""Kernel timeline of one captured c2 training step (CUDA-graph replay,
torch profiler / CUPTI): per-stream busy time, the step span, and the
kernels running while only one stream is busy."""
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

cfg, B = CONFIGS[os.environ.get("CFG", "c4")]()
dev = torch.device("cuda", 0)
model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
opt = FlatAdam(model.P)
Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=1)
st = TrainStep(model, opt, torch.tensor(Xn, device=dev).bfloat16(), [torch.tensor(s, device=dev).bfloat16() for s in Sn],
               [torch.tensor(l, device=dev) for l in Ln], torch.tensor(yn, device=dev)).capture(warmup=3)
for _ in range(3):
    st()
torch.cuda.synchronize()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    st()
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and e.time_range.elapsed_us() > 0]
kern = [(e.time_range.start, e.time_range.end, getattr(e, "device_resource_id", 0), e.name) for e in ev]
kern.sort()
t0, t1 = kern[0][0], max(k[1] for k in kern)
print(f"kernels {len(kern)}, span {(t1 - t0) / 1e3:.3f} ms")
busy = collections.defaultdict(float)
for a, b, s, n in kern:
    busy[s] += b - a
for s, v in sorted(busy.items(), key=lambda x: -x[1]):
    print(f"stream {s}: busy {v / 1e3:.3f} ms")
# time with exactly one / zero kernels running
pts = sorted([(a, 1) for a, b, s, n in kern] + [(b, -1) for a, b, s, n in kern])
cur, last, acc = 0, t0, collections.Counter()
for t, d in pts:
    acc[min(cur, 3)] += t - last
    cur += d
    last = t
print("concurrency histogram (ms):", {k: round(v / 1e3, 3) for k, v in sorted(acc.items())})
# top kernels by time when running alone
alone = collections.Counter()
for a, b, s, n in kern:
    others = sum(1 for a2, b2, s2, n2 in kern if s2 != s and a2 < b and b2 > a)
    if others == 0:
        alone[n[:70]] += b - a
print(f"kernels {len(kern)}, span {(t1 - t0) / 1e3:.3f} ms, alone total {sum(alone.values()) / 1e3:.3f} ms")
for n, v in alone.most_common(25):
    print(f"alone {v / 1e3:7.3f} ms  {n}")
# wall time attributed per kernel name: each instant split evenly over the running kernels
share = collections.Counter()
pts2 = sorted(set([a for a, b, s, n in kern] + [b for a, b, s, n in kern]))
import bisect
for i in range(len(pts2) - 1):
    lo, hi = pts2[i], pts2[i + 1]
    run = [n for a, b, s, n in kern if a <= lo and b >= hi]
    for n in run:
        share[n[:70]] += (hi - lo) / len(run)
print("wall-time share (ms):")
for n, v in share.most_common(30):
    print(f"share {v / 1e3:7.3f} ms  {n}")
