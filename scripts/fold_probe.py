"""Query-fold forward + backward at c2 shapes (4 layers, 32 seeds + 8 CLS,
H=4, d=256), for ncu."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_10016_b200.configs import CONFIGS  # noqa: E402
from paper_2602_10016_b200.model import KunlunModel  # noqa: E402
from paper_2602_10016_b200 import _capi  # noqa: E402

cfg, B = CONFIGS["c2"]()
m = KunlunModel(cfg, torch.device("cuda", 0), torch.bfloat16, seed=0)
if len(sys.argv) > 1:
    _capi.GEMM_LOG = []
for _ in range(3):
    q = m.query_rows()
    loss = sum((v * v).sum() for v in q.values())
    loss.backward()
torch.cuda.synchronize()
if _capi.GEMM_LOG is not None:
    for key, s_, e_ in _capi.GEMM_LOG[-12:]:
        print(f"{s_.elapsed_time(e_) * 1e3:8.1f} us {key}")
