"""PAPER.md Table 2 ablation paths vs the oracle:
``pffn_original`` ("w/o GDPA", gdpa.py:227-257), the PMA-only summary ("w/o
HSP (use PMA)", seqsum.py:26-34), and full attention ("w/o SWA",
attention.py:115-121) — as ops and composed in the model.  The oracle's
ablation functions are pinned to reference outputs
(tests/test_oracle_golden.py::test_pffn_original_golden / test_pma_summary_golden)."""

import numpy as np
import pytest
import torch

from oracle import kunlun as K
from oracle import model as OM
from oracle.parity import grad_errors, rel, relf, violations

pytestmark = pytest.mark.gpu
TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}


@pytest.fixture(autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_10016_b200 import _capi

    _capi.lib()


def _bf(x, dtype):
    return torch.tensor(np.asarray(x)).to(dtype).double().numpy() if dtype == torch.bfloat16 else np.asarray(x)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d", [16, 64])
def test_pffn_original_vs_oracle(dtype, d):
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200 import gdpa as G
    from paper_2602_10016_b200.tensor import Params

    rng = np.random.default_rng(d)
    P = Params()
    pp = G.PffnParams.create(P, "pf", d, 2, d, 2 * d, rng)
    P.finalize("cuda", dtype)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    B, T = 4, 33
    lengths = np.array([T, 7, 0, 1])
    S = _bf(rng.normal(0, 1 / np.sqrt(d), (B, T, d)), dtype)
    Xs = _bf(rng.normal(0, 1, (B, 2, d)), dtype)
    R = rng.normal(0, 1, (B, T, d))
    S_t = torch.tensor(S, dtype=torch.float32, device="cuda", requires_grad=True)
    X_t = torch.tensor(Xs, dtype=torch.float32, device="cuda", requires_grad=True)
    y = G.pffn_original(F.cast(X_t, dtype), F.cast(S_t, dtype), pp, lengths)
    P.zero_grad()
    (F.cast(y, torch.float32) * torch.tensor(R, dtype=torch.float32, device="cuda")).sum().backward()
    err = rel if dtype == torch.float32 else relf
    grads = {}
    for b in range(B):
        L = lengths[b]
        yo, bwd = K.pffn_original(Xs[b], S[b, :L], named, "pf")
        if L:
            assert err(y[b, :L].detach().double().cpu().numpy(), yo) < TOL[dtype]
        assert torch.equal(y[b, L:].detach().float(), F.cast(S_t, dtype).detach()[b, L:].float())  # pass-through
        ds, dx, gr = bwd(R[b, :L])
        for k, v in gr.items():
            K._acc(grads, k, v)
        if L:
            assert err(S_t.grad[b, :L].double().cpu().numpy(), ds) < TOL[dtype]
            assert err(X_t.grad[b].double().cpu().numpy(), dx) < TOL[dtype]
    bad = violations(grad_errors({k: P.grad(k).double().cpu().numpy() for k in grads}, grads, dtype == torch.float32),
                     dtype == torch.float32)
    assert not bad, bad[:6]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d,H", [(32, 2), (256, 4)])
def test_pma_summary_vs_oracle(dtype, d, H):
    from paper_2602_10016_b200 import _capi
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200 import seqsum as Q
    from paper_2602_10016_b200.tensor import Params

    budget = 8
    rng = np.random.default_rng(d + H)
    P = Params()
    sp = Q.SummarizerParams.create(P, "s", d, Q.SummarySplit.for_budget(budget), 6, 2, H, rng, mode="pma")
    P.finalize("cuda", dtype)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    T = 130
    lengths = np.array([T, 0, 57, 1])
    B = len(lengths)
    S = _bf(rng.normal(0, 1, (B, T, d)) * (4.0 / np.sqrt(d) if d > 32 else 1.0), dtype)
    R = rng.normal(0, 1, (B, budget, d))
    S_t = torch.tensor(S, dtype=torch.float32, device="cuda", requires_grad=True)
    _capi.reset_path_hits()
    rows = Q.hsp_summarize(F.cast(S_t, dtype), sp, lengths).rows()
    P.zero_grad()
    (F.cast(rows, torch.float32) * torch.tensor(R, dtype=torch.float32, device="cuda")).sum().backward()
    if dtype == torch.bfloat16 and d == 256:
        assert _capi.path_hits()["hsp_fwd_tc"] > 0  # the fused batch-shared-query pooling
    grads = {}
    for b in range(B):
        L = lengths[b]
        ro, bwd = K.pma_summarize(S[b, :L], named, "s", budget)
        assert rel(rows[b].detach().double().cpu().numpy(), ro) < TOL[dtype]
        ds, gr = bwd(R[b])
        for k, v in gr.items():
            K._acc(grads, k, v)
        if L:
            assert rel(S_t.grad[b, :L].double().cpu().numpy(), ds) < TOL[dtype]
    for k in named:
        grads.setdefault(k, np.zeros_like(named[k]))
    bad = violations(grad_errors({k: P.grad(k).double().cpu().numpy() for k in grads}, grads, dtype == torch.float32),
                     dtype == torch.float32)
    assert not bad, bad[:6]


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("ablation", ["pffn", "pma", "full", "all"])
def test_model_ablation_vs_oracle(dtype, ablation):
    """Composed 2-layer model with the Table 2 switches, parity loss on every output."""
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig

    kw = {"pffn": {"pffn": "original"}, "pma": {"summarizer": "pma"}, "full": {"attention": "full"},
          "all": {"pffn": "original", "summarizer": "pma", "attention": "full"}}[ablation]
    spec = OM.ModelSpec(L=2, d=32, heads=2, n_ctx=5, n_sum=2, n_kv=4, experts=2,
                        events=[OM.EventSpec(T=20, w=3, budget=8, n_seeds=6, rank=2)], **kw)
    cfg = ModelConfig(L=2, d=32, heads=2, n_ctx=5, n_sum=2, n_kv=4, experts=2,
                      events=[EventConfig(T=20, w=3, budget=8, n_seeds=6, rank=2)], **kw)
    pnp = OM.init_params(spec, seed=3)
    model = KunlunModel(cfg, "cuda", dtype)
    assert set(model.P.names()) == set(pnp)
    model.P.load(pnp)
    rng = np.random.default_rng(8)
    B = 3
    lengths = [np.array([20, 6, 0])]
    X = _bf(rng.normal(0, 1 / np.sqrt(32), (B, 5, 32)), dtype)
    S = [_bf(rng.normal(0, 1 / np.sqrt(32), (B, 20, 32)), dtype)]
    labels = np.array([1.0, 0.0, 1.0])
    cot = [{"X": rng.normal(0, 0.1, X.shape), "S": [rng.normal(0, 0.1, S[0].shape)],
            "H": [rng.normal(0, 0.1, (B, 8, 32))]} for _ in range(2)]
    ref = OM.model_forward_backward(spec, pnp, X, S, lengths, labels, cot)
    dv = lambda x, g=False: torch.tensor(np.asarray(x), dtype=torch.float32, device="cuda").requires_grad_(g)
    X_t, S_t = dv(X, True), [dv(S[0], True)]
    logits, outs = model.forward(F.cast(X_t, dtype), [F.cast(S_t[0], dtype)],
                                 [torch.tensor(lengths[0], dtype=torch.int32, device="cuda")],
                                 keep_outputs=True, prune_dead=False)
    loss = F.bce_with_logits(logits, dv(labels))
    for l, (xo, so, ho) in enumerate(outs):
        loss = loss + (F.cast(xo, torch.float32) * dv(cot[l]["X"])).sum()
        loss = loss + (F.cast(so[0], torch.float32) * dv(cot[l]["S"][0])).sum()
        loss = loss + (F.cast(ho[0], torch.float32) * dv(cot[l]["H"][0])).sum()
    model.P.zero_grad()
    loss.backward()
    fp32 = dtype == torch.float32
    errs = {"logits": rel(logits.detach().double().cpu().numpy(), ref["logits"]),
            "dX": (rel if fp32 else relf)(X_t.grad.double().cpu().numpy(), ref["dX"]),
            "dS": (rel if fp32 else relf)(S_t[0].grad.double().cpu().numpy(), ref["dS"][0])}
    for l in range(2):
        errs[f"L{l}/S"] = rel(outs[l][1][0].detach().double().cpu().numpy(), ref["outs"][l]["S"][0])
    gerr = grad_errors({k: model.P.grad(k).double().cpu().numpy() for k in ref["grads"]}, ref["grads"], fp32)
    bad = violations({**errs, **gerr}, fp32)
    assert not bad, bad[:6]
