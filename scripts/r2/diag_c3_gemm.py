"""c3 training step, eager (no graph): every kl_gemm call's shape, operand dtype and
kernel path, with CUDA-event time; summed per (path, shape)."""
import collections, os, sys, torch
sys.path.insert(0, ".")
from paper_2602_10016_b200 import _capi
from paper_2602_10016_b200.configs import CONFIGS
from paper_2602_10016_b200.model import KunlunModel
from paper_2602_10016_b200.optim import FlatAdam, TrainStep
from paper_2602_10016_b200.synth import ctr_batch
from paper_2602_10016_b200 import functional as F

cfg, B = CONFIGS[os.environ.get("CFG", "c3")]()
dev = torch.device("cuda", 0)
model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
opt = FlatAdam(model.P)
Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=1)
X = torch.tensor(Xn, device=dev).bfloat16()
S = [torch.tensor(s, device=dev).bfloat16() for s in Sn]
L = [torch.tensor(l, device=dev) for l in Ln]
if model.groups is not None:
    from paper_2602_10016_b200.grouped import stage
    S, L = stage(S), stage(L)
st = TrainStep(model, opt, X, S, L, torch.tensor(yn, device=dev))
F.BRANCH_STREAMS = False
for _ in range(2):
    st.eager()
torch.cuda.synchronize()
_capi.GEMM_LOG = []
st.eager()
torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for key, s_, e_ in _capi.GEMM_LOG:
    k = (key[:7], key[10], key[14], key[15][-90:])
    agg[k][0] += 1
    agg[k][1] += s_.elapsed_time(e_)
tot = sum(v[1] for v in agg.values())
print(f"gemm calls {len(_capi.GEMM_LOG)}, {tot:.2f} ms (isolated, eager)")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:45]:
    print(f"{v[1]:7.3f} ms n={v[0]:4d} path={k[2]} c={k[1]} MNK..={k[0]} {k[3]}")
