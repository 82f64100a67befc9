import sys, numpy as np, torch
sys.path.insert(0, ".")
from oracle import kunlun as K
from paper_2602_10016_b200 import attention as A, functional as F, _capi
from paper_2602_10016_b200.tensor import Params
for T, w, causal in [(700, 192, False), (700, 255, False), (700, 256, False), (700, 300, False), (700, 383, False), (700, 384, False), (700, 450, False)]:
    d, H = 128, 2
    rng = np.random.default_rng(T + w)
    P = Params(); mp = A.MhaParams.create(P, "m", d, H, rng); P.finalize("cuda", torch.bfloat16)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    lengths = np.array([T, T - 1, 1, 0, max(T // 3, 1)])
    B = len(lengths)
    S = torch.tensor(rng.normal(0, 1, (B, T, d))).bfloat16().double().numpy()
    R = rng.normal(0, 1, (B, T, d))
    S_t = torch.tensor(S, dtype=torch.float32, device="cuda", requires_grad=True)
    _capi.reset_path_hits()
    y = A.mha_window(F.cast(S_t, torch.bfloat16), mp, A.WindowSpec(w, causal), lengths)
    P.zero_grad()
    (F.cast(y, torch.float32) * torch.tensor(R, dtype=torch.float32, device="cuda")).sum().backward()
    torch.cuda.synchronize()
    hits = _capi.path_hits()
    worst = 0.0; wy = 0.0
    for b in range(B):
        L = lengths[b]
        yo, bwd = K.mha_window(S[b, :L], named, "m", w, causal)
        ey = np.abs(y[b, :L].detach().double().cpu().numpy() - yo).max() / max(np.abs(yo).max(), 1e-30) if L else 0
        ds, gr = bwd(R[b, :L])
        eds = np.abs(S_t.grad[b, :L].double().cpu().numpy() - ds).max() / max(np.abs(ds).max(), 1e-30) if L else 0
        worst = max(worst, ey, eds); wy = max(wy, ey)
    print(T, w, causal, "tc fwd/bwd", hits["swa_fwd_tc"], hits["swa_bwd_tc"], "simt", hits["swa_fwd_simt"], "worst rel", f"{worst:.2e}", "fwd", f"{wy:.2e}", flush=True)
