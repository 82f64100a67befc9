"""Grouped event types (grouped.py; north_star (1) "event-level
personalization executed as a grouped GEMM over event types").

* the grouped path and the per-event path (``group_events=False``) on the
  same parameters and inputs agree (device vs device, bf16 at the c3 widths
  d=256 / H=4 / w=128 with CompSkip, and fp32 at toy widths), and the
  grouped path launches far fewer kernels;
* fp32 grouped vs the float64 oracle within 1e-5 (the GEMM-composition
  pooling with one query set per event group);
* kl_hsp_fwd/bwd with q_group: per-group query sets equal separate launches.
The bf16 oracle comparison of the grouped path is
test_gpu_model_parity.py's "grouped" cases."""

import numpy as np
import pytest
import torch

from oracle import model as OM
from oracle.parity import grad_errors, rel, violations

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_10016_b200 import _capi

    _capi.lib()


def _pair(dtype, d, heads, T, w, budget, seeds, rank, E, L=2, compskip=False, n_ctx=16):
    from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig

    ms = []
    for grp in (True, False):
        ev = [EventConfig(T=T, w=w, budget=budget, n_seeds=seeds, rank=rank) for _ in range(E)]
        cfg = ModelConfig(L=L, d=d, heads=heads, n_ctx=n_ctx, events=ev, compskip=compskip, group_events=grp)
        ms.append(KunlunModel(cfg, "cuda", dtype, seed=3))
    assert ms[0].groups is not None and ms[1].groups is None
    return ms


def _run(model, X, S, L, y):
    from paper_2602_10016_b200 import _capi
    from paper_2602_10016_b200 import functional as F

    model.P.zero_grad()
    n0 = _capi.launch_count()
    loss, logits = model.loss(X, S, L, y)
    loss.backward()
    torch.cuda.synchronize()
    return logits.detach().double().cpu().numpy(), model.P.gflat.detach().double().cpu().numpy(), \
        _capi.launch_count() - n0


@pytest.mark.parametrize("compskip", [False, True])
def test_grouped_equals_per_event_bf16(compskip):
    from paper_2602_10016_b200.synth import ctr_batch

    g, p = _pair(torch.bfloat16, 256, 4, 512, 128, 8, 8, 2, E=4, L=4, compskip=compskip)
    Xn, Sn, Ln, yn = ctr_batch(g.cfg, 6, seed=5, full_length=False)
    dev = lambda a, dt=torch.bfloat16: torch.tensor(a, device="cuda").to(dt)
    X, S, L, y = dev(Xn), [dev(s) for s in Sn], [torch.tensor(l, device="cuda") for l in Ln], dev(yn, torch.float32)
    zg, gg, ng = _run(g, X, S, L, y)
    zp, gp, np_ = _run(p, X, S, L, y)
    assert rel(zg, zp) < 1e-2, rel(zg, zp)
    assert np.linalg.norm(gg - gp) / np.linalg.norm(gp) < 2e-2
    # every block's gradient, per registry name
    bad = [(n, e) for n in g.P.names()
           for e in [np.linalg.norm(g.P.grad(n).double().cpu().numpy() - p.P.grad(n).double().cpu().numpy())
                     / max(np.linalg.norm(p.P.grad(n).double().cpu().numpy()), 1e-30)] if e > 5e-2]
    assert not bad, bad[:6]
    assert ng < 0.7 * np_, (ng, np_)  # one launch per operator instead of one per event type (E = 4 here)


def test_grouped_fp32_vs_oracle():
    """fp32 grouped path (composition pooling with per-event query sets,
    SIMT attention) vs the oracle at 1e-5."""
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig

    E, D, T = 3, 32, 11
    evs = [dict(T=T, w=3, budget=8, n_seeds=6, rank=2) for _ in range(E)]
    spec = OM.ModelSpec(L=2, d=D, heads=4, n_ctx=5, n_sum=2, n_kv=4, experts=2,
                        events=[OM.EventSpec(**e) for e in evs])
    cfg = ModelConfig(L=2, d=D, heads=4, n_ctx=5, n_sum=2, n_kv=4, experts=2, events=[EventConfig(**e) for e in evs])
    pnp = OM.init_params(spec, seed=9)
    model = KunlunModel(cfg, "cuda", torch.float32)
    assert model.groups is not None
    model.P.load(pnp)
    rng = np.random.default_rng(4)
    B = 3
    lengths = [np.array([T, 5, 0]), np.array([1, T, 7]), np.array([0, 2, T])]
    X = rng.normal(0, 0.2, (B, 5, D))
    S = [rng.normal(0, 0.2, (B, T, D)) for _ in range(E)]
    labels = np.array([1.0, 0.0, 1.0])
    cot = [{"X": rng.normal(0, 0.1, X.shape), "S": [rng.normal(0, 0.1, s.shape) for s in S],
            "H": [rng.normal(0, 0.1, (B, 8, D)) for _ in range(E)]} for _ in range(2)]
    ref = OM.model_forward_backward(spec, pnp, X, S, lengths, labels, cot)
    dv = lambda x, g=False: torch.tensor(np.asarray(x), dtype=torch.float32, device="cuda").requires_grad_(g)
    X_t, S_t = dv(X, True), [dv(s, True) for s in S]
    logits, outs = model.forward(X_t, S_t, [torch.tensor(L, dtype=torch.int32, device="cuda") for L in lengths],
                                 keep_outputs=True, prune_dead=False)
    loss = F.bce_with_logits(logits, dv(labels))
    for l, (xo, so, ho) in enumerate(outs):
        loss = loss + (xo * dv(cot[l]["X"])).sum()
        for e in range(E):
            loss = loss + (so[e] * dv(cot[l]["S"][e])).sum() + (ho[e] * dv(cot[l]["H"][e])).sum()
    model.P.zero_grad()
    loss.backward()
    errs = {"logits": rel(logits.detach().double().cpu().numpy(), ref["logits"]),
            "dX": rel(X_t.grad.double().cpu().numpy(), ref["dX"])}
    for e in range(E):
        errs[f"dS{e}"] = rel(S_t[e].grad.double().cpu().numpy(), ref["dS"][e])
        for l in range(2):
            errs[f"L{l}/S{e}"] = rel(outs[l][1][e].detach().double().cpu().numpy(), ref["outs"][l]["S"][e])
            errs[f"L{l}/H{e}"] = rel(outs[l][2][e].detach().double().cpu().numpy(), ref["outs"][l]["H"][e])
    gerr = grad_errors({k: model.P.grad(k).double().cpu().numpy() for k in ref["grads"]}, ref["grads"], True)
    bad = violations({**errs, **gerr}, True, set())
    assert not bad, bad[:6]


@pytest.mark.parametrize("d", [256, 512])
def test_hsp_q_group_equals_separate_launches(d, monkeypatch):
    """kl_hsp_fwd / kl_hsp_bwd with q_group (one query set per group of
    samples) == one launch per group with its own set (bf16, fused kernels).
    d = 512: one CTA per (group, query tile, half) lane (KL_HSP_CPL=1), so
    both launches pool every sample whole and agree bitwise (the balanced
    split is checked against the composition in test_gpu_parity)."""
    from paper_2602_10016_b200 import functional as F

    monkeypatch.setenv("KL_HSP_CPL", "1")

    torch.manual_seed(0)
    G, Bg, T, HQ = 3, 4, 300, 40
    S = (torch.randn(G * Bg, T, d, device="cuda") / d ** 0.5).to(torch.bfloat16)
    Q = torch.randn(G, HQ, d, device="cuda") * 0.5
    lens = torch.randint(0, T + 1, (G * Bg,), device="cuda", dtype=torch.int32)
    lens[0], lens[5] = 0, T
    gO = [torch.randn(G * Bg, n, d, device="cuda").to(torch.bfloat16) for n in (32, 8)]
    S1, Q1 = S.clone().requires_grad_(True), Q.clone().requires_grad_(True)
    o1 = F.hsp_pool(S1, Q1, lens, (32, 8))
    (sum((o.float() * g.float()).sum() for o, g in zip(o1, gO))).backward()
    for gi in range(G):
        sl = slice(gi * Bg, (gi + 1) * Bg)
        S2, Q2 = S[sl].clone().requires_grad_(True), Q[gi].clone().requires_grad_(True)
        o2 = F.hsp_pool(S2, Q2, lens[sl], (32, 8))
        (sum((o.float() * g[sl].float()).sum() for o, g in zip(o2, gO))).backward()
        for a, b in zip(o1, o2):
            assert torch.equal(a[sl], b)
        assert torch.equal(S1.grad[sl], S2.grad)
        assert rel(Q1.grad[gi].double().cpu().numpy(), Q2.grad.double().cpu().numpy()) < 1e-5
