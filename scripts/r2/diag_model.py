"""Diagnose model-level bf16 parity at the tcgen05 shapes under kernel toggles."""
import sys, itertools
import numpy as np, torch
sys.path.insert(0, ".")
from oracle import model as OM
from oracle.parity import grad_errors, rel, relf
from paper_2602_10016_b200 import _capi, functional as F
from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig

def run(events, lengths, toggles, L=2, compskip=False, B=5, seed=21):
    spec = OM.ModelSpec(L=L, d=256, heads=4, n_ctx=16, n_sum=4, n_kv=16, experts=2, compskip=compskip,
                        events=[OM.EventSpec(**e) for e in events])
    pnp = OM.init_params(spec, seed=seed)
    cfg = ModelConfig(L=L, d=256, heads=4, n_ctx=16, n_sum=4, n_kv=16, experts=2, compskip=compskip,
                      events=[EventConfig(**e) for e in events])
    rng = np.random.default_rng(7)
    bf = lambda x: torch.tensor(x).to(torch.bfloat16).double().numpy()
    X = bf(rng.normal(0, 1 / 16, (B, 16, 256)))
    S = [bf(rng.normal(0, 1 / 16, (B, e["T"], 256))) for e in events]
    labels = (rng.random(B) < 0.4).astype(np.float64)
    cot = [{"X": rng.normal(0, 0.05, X.shape), "S": [rng.normal(0, 0.05, s.shape) for s in S],
            "H": [rng.normal(0, 0.05, (B, e["budget"], 256)) for e in events]} for _ in range(L)]
    ref = OM.model_forward_backward(spec, pnp, X, S, lengths, labels, cot)
    for tog in toggles:
        for k, v in tog.items():
            setattr(F, k, v)
        model = KunlunModel(cfg, "cuda", torch.bfloat16)
        model.P.load(pnp)
        dev = lambda x, g=False: torch.tensor(np.asarray(x), dtype=torch.float32, device="cuda").requires_grad_(g)
        X_t = dev(X, True); S_t = [dev(s, True) for s in S]
        lens = [torch.tensor(l, dtype=torch.int32, device="cuda") for l in lengths]
        _capi.reset_path_hits()
        logits, outs = model.forward(F.cast(X_t, torch.bfloat16), [F.cast(s, torch.bfloat16) for s in S_t], lens,
                                     keep_outputs=True, prune_dead=False)
        loss = F.bce_with_logits(logits, dev(labels))
        for l, (xo, so, ho) in enumerate(outs):
            loss = loss + (F.cast(xo, torch.float32) * dev(cot[l]["X"])).sum()
            for e in range(len(events)):
                loss = loss + (F.cast(so[e], torch.float32) * dev(cot[l]["S"][e])).sum()
                loss = loss + (F.cast(ho[e], torch.float32) * dev(cot[l]["H"][e])).sum()
        model.P.zero_grad()
        loss.backward()
        torch.cuda.synchronize()
        errs = {"logits": rel(logits.detach().double().cpu().numpy(), ref["logits"])}
        for l in range(L):
            xo, so, ho = outs[l]
            errs[f"L{l}/X"] = rel(xo.detach().double().cpu().numpy(), ref["outs"][l]["X"])
            for e in range(len(events)):
                errs[f"L{l}/S{e}"] = rel(so[e].detach().double().cpu().numpy(), ref["outs"][l]["S"][e])
                errs[f"L{l}/H{e}"] = rel(ho[e].detach().double().cpu().numpy(), ref["outs"][l]["H"][e])
        errs["dX"] = relf(X_t.grad.double().cpu().numpy(), ref["dX"])
        for e in range(len(events)):
            g = S_t[e].grad.double().cpu().numpy()
            errs[f"dS{e}"] = relf(g, ref["dS"][e])
            for b in range(B):
                errs[f"dS{e}[b{b},len{lengths[e][b]}]"] = relf(g[b], ref["dS"][e][b])
        gerr = grad_errors({k: model.P.grad(k).double().cpu().numpy() for k in ref["grads"]}, ref["grads"], False)
        allr = sorted(list(errs.items()) + list(gerr.items()), key=lambda kv: -kv[1])
        hits = {k: v for k, v in _capi.path_hits().items() if v}
        print(f"== events={[(e['T'], e['budget']) for e in events]} lengths={[list(l) for l in lengths]} tog={tog} L={L} cs={compskip}")
        print("   hits", hits)
        print("   worst:", ", ".join(f"{k}={v:.2e}" for k, v in allr[:10]))
        for k, v in tog.items():
            setattr(F, k, True)

E0 = dict(T=1024, w=128, budget=32, n_seeds=32, rank=8)
E1 = dict(T=384, w=128, budget=8, n_seeds=8, rank=2)
T0 = [{}, {"HSP_FUSED": False}, {"GDPA_FUSED": False}, {"BRANCH_STREAMS": False}]
run([E1], [np.array([384, 384, 384, 384, 384])], T0, L=1)
run([E1], [np.array([384, 0, 383, 129, 1])], T0, L=1)
run([E0, E1], [np.array([1024, 1023, 129, 1, 0]), np.array([384, 0, 383, 129, 1])], T0, L=2)
