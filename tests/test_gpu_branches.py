"""Parallel stream branches (the layer's summary / interaction branch beside
the sequence branch, the Wukong experts beside each other; CUDA-graph fork /
join when captured) must give the same loss and gradients as the serial
issue order: a missing cross-stream dependency shows up as a lost gradient
contribution or a stale read, far outside the bf16 tolerance used here."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _run(model, batch, graph):
    from paper_2602_10016_b200.optim import FlatAdam, TrainStep

    X, S, L, y = batch
    if not graph:
        model.P.zero_grad()
        loss, logits = model.loss(X, S, L, y)
        loss.backward()
        torch.cuda.synchronize()
        return float(loss), logits.detach().float().clone(), model.P.gflat.detach().clone()
    opt = FlatAdam(model.P, lr=0.0)
    st = TrainStep(model, opt, X, S, L, y)
    if graph == "eager-step":  # TrainStep without capture (weight-gradient stream on)
        st.loss = st.eager()
    else:
        st.capture(warmup=1)
        model.P.zero_grad()
        st()
    torch.cuda.synchronize()
    return float(st.loss.detach()), None, model.P.gflat.detach().clone()


@pytest.mark.parametrize("compskip", [False, True])
def test_branch_streams_match_serial(compskip):
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig
    from paper_2602_10016_b200.synth import ctr_batch

    cfg = ModelConfig(L=3, d=256, heads=4, n_ctx=16, compskip=compskip,
                      events=[EventConfig(T=384, w=128, budget=32, n_seeds=32, rank=8)])
    dev = torch.device("cuda", 0)
    model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
    Xn, Sn, Ln, yn = ctr_batch(cfg, 8, seed=3)
    Ln = [np.array([384, 200, 1, 0, 384, 383, 129, 64], dtype=np.int32)]
    batch = (torch.tensor(Xn, device=dev).bfloat16(), [torch.tensor(s, device=dev).bfloat16() for s in Sn],
             [torch.tensor(l, device=dev) for l in Ln], torch.tensor(yn, device=dev))
    old = F.BRANCH_STREAMS
    try:
        F.BRANCH_STREAMS = False
        l0, z0, g0 = _run(model, batch, graph=False)
        F.BRANCH_STREAMS = True
        l1, z1, g1 = _run(model, batch, graph=False)
        l2, _, g2 = _run(model, batch, graph=True)
        l3, _, g3 = _run(model, batch, graph="eager-step")
    finally:
        F.BRANCH_STREAMS = old
    scale = float(g0.abs().max())
    assert abs(l1 - l0) <= 1e-3 * max(1.0, abs(l0))
    assert float((z1 - z0).abs().max()) <= 1e-2 * max(1.0, float(z0.abs().max()))
    assert float((g1 - g0).abs().max()) <= 2e-2 * scale
    assert abs(l2 - l0) <= 1e-3 * max(1.0, abs(l0))
    assert float((g2 - g0).abs().max()) <= 2e-2 * scale
    assert abs(l3 - l0) <= 1e-3 * max(1.0, abs(l0))
    assert float((g3 - g0).abs().max()) <= 2e-2 * scale


def test_split_adam_matches_single():
    """Adam split by layer (launched from the layer boundaries beside the
    remaining backward, query-fold inputs last) applies exactly the Adam
    update to every parameter, from the step's final gradients: checked
    against a torch restatement of the update on the same gradients, over
    three steps (m, v and the device step count carried)."""
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig
    from paper_2602_10016_b200.optim import FlatAdam, TrainStep
    from paper_2602_10016_b200.synth import ctr_batch

    cfg = ModelConfig(L=3, d=256, heads=4, n_ctx=16, compskip=True,
                      events=[EventConfig(T=256, w=64, budget=32, n_seeds=32, rank=8)])
    dev = torch.device("cuda", 0)
    Xn, Sn, Ln, yn = ctr_batch(cfg, 8, seed=5)
    old = F.BRANCH_STREAMS
    try:
        F.BRANCH_STREAMS = True
        model = KunlunModel(cfg, dev, torch.bfloat16, seed=0)
        batch = (torch.tensor(Xn, device=dev).bfloat16(), [torch.tensor(s, device=dev).bfloat16() for s in Sn],
                 [torch.tensor(l, device=dev) for l in Ln], torch.tensor(yn, device=dev))
        opt = FlatAdam(model.P, lr=1e-3)
        st = TrainStep(model, opt, *batch[:3], batch[3])
        assert st.segments is not None
        for step in range(1, 4):
            p0, m0, v0 = model.P.flat.detach().clone(), opt.m.clone(), opt.v.clone()
            st.eager()
            torch.cuda.synchronize()
            g = model.P.gflat.detach()
            m1 = opt.b1 * m0 + (1 - opt.b1) * g
            v1 = opt.b2 * v0 + (1 - opt.b2) * g * g
            ref = p0 - opt.lr * (m1 / (1 - opt.b1 ** step)) / ((v1 / (1 - opt.b2 ** step)).sqrt() + opt.eps)
            assert int(opt.t.item()) == step
            assert float((opt.m - m1).abs().max()) <= 1e-6 * max(1e-30, float(m1.abs().max()))
            assert float((model.P.flat.detach() - ref).abs().max()) <= 1e-6
            # the bf16 compute mirror follows the masters
            assert float((model.P.flat_c.float() - model.P.flat.detach()).abs().max()) <= 1e-2
    finally:
        F.BRANCH_STREAMS = old
