"""Preprocessing on the device vs the oracle (pinned to the reference's
preproc outputs, tests/test_oracle_golden.py::test_preproc_golden):
``embed_nonseq`` (embed_dense + embed_sparse + assemble_nonseq fused into one
gather kernel, scatter-add VJP), ``fuse_sequences`` over right-aligned
sequences, the schemas' validation and IndexError contract."""

import numpy as np
import pytest
import torch

from oracle import ops
from oracle.parity import rel, relf

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("d,m,vocabs,B", [(8, 3, [5, 7, 2], 4), (256, 13, [1000, 17, 3, 50000], 64)])
def test_embed_nonseq_vs_oracle(dtype, d, m, vocabs, B):
    from paper_2602_10016_b200 import _capi
    from paper_2602_10016_b200.preproc import EventSchema, FeatureSchema, NonSeqEmbeddingParams, embed_nonseq
    from paper_2602_10016_b200.tensor import Params

    schema = FeatureSchema(m, vocabs, [EventSchema("click", 10, 8)], d)
    rng = np.random.default_rng(d + B)
    P = Params()
    emb = NonSeqEmbeddingParams.create(P, "emb", schema, rng)
    P.finalize("cuda", dtype)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    x = rng.normal(0, 1, (B, m)).astype(np.float32)
    ids = np.stack([rng.integers(0, v, B) for v in vocabs], axis=1)
    ids[0] = 0
    ids[1] = np.array(vocabs) - 1  # both ends of every vocabulary
    if B > 4:
        ids[2:6, 0] = 7  # repeated ids: the VJP's atomics accumulate
    out = embed_nonseq(x, ids, emb)
    assert out.shape == (B, len(vocabs) + 1, d) and out.dtype == dtype
    g = rng.normal(0, 1, out.shape)
    P.zero_grad()
    out.backward(torch.tensor(g, device="cuda", dtype=dtype))
    torch.cuda.synchronize()
    gq = torch.tensor(g).to(dtype).double().numpy()
    tabs = [named[f"emb/sparse{i}"] for i in range(len(vocabs))]
    dproj = np.zeros_like(named["emb/dense_proj"])
    dts = [np.zeros_like(t) for t in tabs]
    err = rel if dtype == torch.float32 else relf
    tol = 1e-5 if dtype == torch.float32 else 2e-2
    for b in range(B):
        o, bwd = ops.embed_nonseq(x[b].astype(np.float64), ids[b], named["emb/dense_proj"], tabs)
        assert err(out[b].detach().double().cpu().numpy(), o) < tol
        # gathered rows are copies: bit-exact against the (compute-dtype) table rows
        for i in range(len(vocabs)):
            assert torch.equal(out[b, 1 + i], P.w(emb.tables)[emb.offsets[i] + ids[b, i]])
        dp, dt = bwd(gq[b])
        dproj += dp
        for i in range(len(vocabs)):
            dts[i] += dt[i]
    assert err(P.grad("emb/dense_proj").double().cpu().numpy(), dproj) < tol
    for i in range(len(vocabs)):
        assert rel(P.grad(f"emb/sparse{i}").double().cpu().numpy(), dts[i]) < 1e-5  # fp32 atomics of bf16 rows
    with pytest.raises(IndexError):
        bad = ids.copy()
        bad[0, 0] = vocabs[0]
        embed_nonseq(x, bad, emb)


def test_fuse_sequences_and_align_right_vs_oracle():
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200.mlp import Mlp
    from paper_2602_10016_b200.preproc import align_right, fuse_sequences
    from paper_2602_10016_b200.tensor import Params, ShapeError

    d, K_, T = 16, 3, 9
    rng = np.random.default_rng(2)
    P = Params()
    fusion = Mlp.create(P, "fus", [K_ * d, 24, d], ["silu", "identity"], rng)
    P.finalize("cuda", torch.float32)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    raw = [rng.normal(0, 1, (t, d)) for t in (4, 9, 1)]
    al = align_right(raw, T)
    al_t = align_right([torch.tensor(r, device="cuda") for r in raw], T)
    for a, at in zip(al, al_t):
        assert np.array_equal(a, at.cpu().numpy())
    seqs = [torch.tensor(a, dtype=torch.float32, device="cuda", requires_grad=True) for a in al]
    y = fuse_sequences(seqs, fusion)
    g = rng.normal(0, 1, y.shape)
    y.backward(torch.tensor(g, dtype=torch.float32, device="cuda"))
    yo, bwd = ops.fuse_sequences(al, [named["fus/w0"], named["fus/w1"]], [named["fus/b0"], named["fus/b1"]],
                                 ["silu", "identity"])
    assert rel(y.detach().double().cpu().numpy(), yo) < 1e-5
    dseqs, _, _ = bwd(g)
    for s, ds in zip(seqs, dseqs):
        assert rel(s.grad.double().cpu().numpy(), ds) < 1e-5
    with pytest.raises(ShapeError):
        align_right(raw, 3)
    with pytest.raises(ShapeError):
        fuse_sequences([seqs[0], seqs[1][:4]], fusion)
