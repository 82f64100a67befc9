"""Timing probe of kl_rote (the ROTE kernel) at a c4-sized batch:
    python scripts/probes/rote_probe.py [B T d] [iters]
Prints device time per launch (CUDA events, inputs >> L2 rotate through 4
buffers) and achieved algorithmic HBM bandwidth: read x + write y (bf16) +
read the fp64 timestamps."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2602_10016_b200.preproc import RoteConfig, rote_sequence  # noqa: E402

B, T, d = (int(x) for x in sys.argv[1:4]) if len(sys.argv) > 3 else (32, 4096, 512)
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20
cfg = RoteConfig.default(d)
xs = [torch.randn(B, T, d, device="cuda").bfloat16() for _ in range(4)]
ts = torch.cumsum(torch.rand(B, T, device="cuda", dtype=torch.float64) * 600, 1)
lens = torch.full((B,), T, device="cuda", dtype=torch.int32)
for i in range(3):
    rote_sequence(xs[i % 4], ts, cfg, lengths=lens)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for i in range(iters):
    rote_sequence(xs[i % 4], ts, cfg, lengths=lens)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / iters
byt = 2 * B * T * d * 2 + B * T * 8
print(f"kl_rote B={B} T={T} d={d}: {ms * 1e3:.1f} us/launch (incl. output allocation), {byt / ms / 1e6:.0f} GB/s algorithmic")
