"""Pin the numpy oracle against golden vectors produced by the unmodified
reference (tests/golden/make_golden.py).  CPU only."""

import os

import numpy as np
import pytest

from oracle import kunlun as K
from oracle import model as OM

G = os.path.join(os.path.dirname(__file__), "golden")
TOL = 1e-10


def load(name):
    z = np.load(os.path.join(G, name))
    params = {k[6:]: z[k] for k in z.files if k.startswith("param:")}
    grads = {k[5:]: z[k] for k in z.files if k.startswith("grad:")}
    return z, params, grads


def rel(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = max(np.abs(b).max() if b.size else 0.0, 1e-300)
    return (np.abs(a - b).max() if b.size else 0.0) / den


@pytest.mark.parametrize("tag", ["default", "sigexp"])
def test_gdpa(tag):
    z, p, g = load(f"gdpa_{tag}.npz")
    d, H, n_kv, n_sum, n_ctx, t_len = z["meta"]
    acts = [str(a) for a in z["acts"]]
    s, x, pool = p["in/S"], p["in/X"], p["pool"]
    xs, xs_bwd = K.summarize_nonseq(x, pool)
    kv, kv_bwd = K.generate_kv(xs, p, "g", int(n_kv))
    y, y_bwd = K.gdpa_forward(s, kv, p, "g", float(t_len), acts)
    assert rel(y, z["out_Y"]) < TOL
    ds, dkvs, gr = y_bwd(z["cot_Y"])
    dxs, gr2 = kv_bwd(dkvs)
    dx, dpool = xs_bwd(dxs)
    gr.update(gr2)
    gr["in/S"], gr["in/X"], gr["pool"] = ds, dx, dpool
    for k, v in g.items():
        assert rel(gr[k], v) < TOL, k


@pytest.mark.parametrize("tag", ["w3_len9", "w3_causal", "full_len7", "w0_len0"])
def test_mha(tag):
    z, p, g = load(f"mha_{tag}.npz")
    d, H, t_len, w, causal, length, full = z["meta"]
    length = None if length < 0 else int(length)
    s = p["in/S"]
    if full:
        y, bwd = K.mha_full(s, p, "m", length)
    else:
        y, bwd = K.mha_window(s, p, "m", int(w), bool(causal), length)
    assert rel(y, z["out_Y"]) < TOL
    ds, gr = bwd(z["cot_Y"])
    gr["in/S"] = ds
    for k, v in g.items():
        assert rel(gr[k], v) < TOL, k


@pytest.mark.parametrize("tag", ["t10", "t1", "t0"])
def test_hsp(tag):
    z, p, g = load(f"hsp_{tag}.npz")
    d, H, t_len, budget, n_seeds, rank = z["meta"]
    rows, bwd = K.hsp_summarize(p["in/S"], p, "s", int(budget))
    assert rel(rows, z["out_Y"]) < TOL
    ds, gr = bwd(z["cot_Y"])
    gr["in/S"] = ds
    for k, v in g.items():
        got = gr.get(k, np.zeros_like(v))
        assert rel(got, v) < TOL or np.abs(v).max() == np.abs(got).max() == 0, k


def test_gi():
    z, p, g = load("gi.npz")
    d, n_ctx, experts, hidden, *budgets = z["meta"]
    rows = [p[f"in/R{e}"] for e in range(len(budgets))]
    y, bwd = K.global_interaction(p["in/X"], rows, p, "gi", int(experts))
    assert rel(y, z["out_Y"]) < TOL
    dx, drows, gr = bwd(z["cot_Y"])
    gr["in/X"] = dx
    for e, dr in enumerate(drows):
        gr[f"in/R{e}"] = dr
    for k, v in g.items():
        assert rel(gr[k], v) < TOL, k


def _model_spec(compskip):
    return OM.ModelSpec(L=2, d=16, heads=4, n_ctx=5, n_sum=2, n_kv=4, experts=2, compskip=compskip,
                        events=[OM.EventSpec(T=12, w=3, budget=8, n_seeds=6, rank=2),
                                OM.EventSpec(T=9, w=2, budget=4, n_seeds=3, rank=1)])


@pytest.mark.parametrize("tag,compskip", [("noskip", False), ("compskip", True)])
def test_model(tag, compskip):
    z, p, g = load(f"model_{tag}.npz")
    spec = _model_spec(compskip)
    S = [z["S0"], z["S1"]]
    lengths = [z["len0"], z["len1"]]
    cot = [{"X": z[f"cot{l}_X"], "S": [z[f"cot{l}_S{e}"] for e in range(2)],
            "H": [z[f"cot{l}_H{e}"] for e in range(2)]} for l in range(spec.L)]
    r = OM.model_forward_backward(spec, p, z["X"], S, lengths, z["labels"], cot)
    # the oracle's parity loss also covers padding rows (identity outputs);
    # the reference sees only valid rows, so remove that constant term.
    pad = sum(float((S[e][b, lengths[e][b]:] * cot[l]["S"][e][b, lengths[e][b]:]).sum())
              for l in range(spec.L) for e in range(2) for b in range(S[e].shape[0]))
    assert abs(r["loss"] - pad - float(z["loss"])) < 1e-10 * max(1.0, abs(float(z["loss"])))
    assert rel(r["logits"], z["logits"]) < TOL
    assert rel(r["dX"], z["dX"]) < TOL
    for e in range(2):
        assert rel(r["dS"][e], z[f"dS{e}"]) < TOL
    for k, v in g.items():
        assert rel(r["grads"][k], v) < TOL or (np.abs(v).max() == 0 and np.abs(r["grads"][k]).max() == 0), k


def test_index_kats():
    z = np.load(os.path.join(G, "index.npz"))
    for k in z.files:
        parts = k.split("_")
        if parts[0] == "band":
            t, w, c = map(int, parts[1:])
            assert np.array_equal(K.band_mask(t, w, bool(c)), z[k])
        elif parts[0] == "support":
            t, w, c = map(int, parts[1:])
            assert np.array_equal(K.band_support_sizes(t, w, bool(c)), z[k])
        elif parts[0] == "experts":
            tot, m = map(int, parts[1:])
            assert np.array_equal(np.array(K.expert_ranges(tot, m)), z[k])
        elif parts[0] == "split":
            assert list(K.split_for_budget(int(parts[1]))) == list(z[k])


def test_compskip_spec_examples():
    # SPEC.md:480-482
    assert OM.compskip_config(4) == [(True, False, False), (False, True, True)] * 2
    assert OM.compskip_config(1) == [(True, False, False)]
    assert OM.compskip_config(3, enabled=False) == [(False, False, False)] * 3
    with pytest.raises(ValueError):
        OM.compskip_config(0)


def test_normalized_entropy_spec_examples():
    """SPEC.md:559-561 examples and the SPEC.md:557 error contract."""
    from oracle import ops

    eps = 1e-12
    assert abs(ops.normalized_entropy([1, 0, 1, 0], [0.5] * 4)["ne"] - 1.0) < 1e-12
    assert ops.normalized_entropy([1, 0], [1 - eps, eps])["ne"] < 1e-10
    r = ops.normalized_entropy([1, 0, 0, 0], [0.7, 0.1, 0.1, 0.1])
    assert abs(r["ne"] - 0.2991) < 5e-5 and r["ctr"] == 0.25 and r["n"] == 4
    assert abs(r["ne"] - r["cross_entropy"] / r["background_entropy"]) < 1e-15
    z = np.random.default_rng(0).normal(size=64) * 4
    y = (np.arange(64) % 3 == 0).astype(np.float64)
    a = ops.normalized_entropy(y, z, from_logits=True)["ne"]
    b = ops.normalized_entropy(y, 1 / (1 + np.exp(-z)))["ne"]
    assert abs(a - b) < 1e-12
    for bad in ([0, 0, 0], [1, 1]):
        with pytest.raises(ValueError, match="degenerate background entropy"):
            ops.normalized_entropy(bad, [0.5] * len(bad))


@pytest.mark.parametrize("tag", ["prev", "latest", "nots", "custom", "empty"])
def test_rote(tag):
    """oracle.ops.rote_sequence vs the reference's rote_sequence (preproc.py:187-199)."""
    from oracle import ops

    z = np.load(os.path.join(G, "rote.npz"))
    ts = z[f"{tag}:ts"] if int(z[f"{tag}:has_ts"]) else None
    y, bwd = ops.rote_sequence(z[f"{tag}:S"], ts, z[f"{tag}:pos"], z[f"{tag}:temp"], float(z[f"{tag}:tau_scale"]),
                               "previous" if int(z[f"{tag}:mode"]) == 0 else "latest")
    assert y.shape == z[f"{tag}:Y"].shape
    assert rel(y, z[f"{tag}:Y"]) < 1e-12
    assert rel(bwd(z[f"{tag}:cot"]), z[f"{tag}:dS"]) < 1e-12


@pytest.mark.parametrize("T,w,causal,length", [(300, 17, False, 300), (300, 128, True, 257), (129, 0, False, 1),
                                               (260, 200, False, 0)])
def test_banded_mha_equals_dense(T, w, causal, length):
    """The oracle's block-banded mha_window (used above T = 1024) is the dense
    masked evaluation (the reference's own, attention.py:69-129) with the
    exactly-masked entries skipped: outputs and VJPs agree to float64
    rounding."""
    from oracle import kunlun as K
    from oracle import model as OM

    spec = OM.ModelSpec(L=1, d=32, heads=4, n_ctx=2, events=[OM.EventSpec(T=T, w=w, budget=4, n_seeds=4, rank=1)])
    p = OM.init_params(spec, seed=3)
    rng = np.random.default_rng(T + w)
    s = rng.normal(0, 1, (T, 32))
    g = rng.normal(0, 1, (T, 32))
    yd, bd = K.mha_window(s, p, "L0/ev0/mha", w, causal, length, banded=False)
    yb, bb = K.mha_window(s, p, "L0/ev0/mha", w, causal, length, banded=True)
    assert np.abs(yd - yb).max() <= 1e-12 * max(1.0, np.abs(yd).max())
    (dd, gd), (db, gb) = bd(g), bb(g)
    assert np.abs(dd - db).max() <= 1e-12 * max(1.0, np.abs(dd).max())
    for k in gd:
        assert np.abs(gd[k] - gb[k]).max() <= 1e-12 * max(1.0, np.abs(gd[k]).max()), k


def test_pffn_original_golden():
    """oracle.kunlun.pffn_original vs the reference's gdpa.pffn_original (Table 2 'w/o GDPA')."""
    from oracle import kunlun as K

    z = np.load(os.path.join(G, "pffn_original.npz"))
    p = {k[len("param:"):]: z[k] for k in z.files if k.startswith("param:")}
    g = {k[len("grad:"):]: z[k] for k in z.files if k.startswith("grad:")}
    y, bwd = K.pffn_original(p["in/Xsum"], p["in/S"], p, "pf")
    assert np.abs(y - z["out_Y"]).max() < 1e-10
    ds, dx, gr = bwd(z["cot_Y"])
    assert np.abs(ds - g["in/S"]).max() < 1e-10
    assert np.abs(dx - g["in/Xsum"]).max() < 1e-10
    for k, v in gr.items():
        assert np.abs(v - g[k]).max() < 1e-10, k


@pytest.mark.parametrize("tag", ["t10", "t0"])
def test_pma_summary_golden(tag):
    """oracle.kunlun.pma_summarize vs [pma(CLS) | pma(Q_learn) | recent] run on the reference (Table 2 'w/o HSP')."""
    from oracle import kunlun as K

    z = np.load(os.path.join(G, f"pma_summary_{tag}.npz"))
    p = {k[len("param:"):]: z[k] for k in z.files if k.startswith("param:")}
    g = {k[len("grad:"):]: z[k] for k in z.files if k.startswith("grad:")}
    d, H, budget, t_len = (int(v) for v in z["meta"])
    rows, bwd = K.pma_summarize(p["in/S"], p, "s", budget)
    assert np.abs(rows - z["out_rows"]).max() < 1e-10
    ds, gr = bwd(z["cot"])
    if t_len:
        assert np.abs(ds - g["in/S"]).max() < 1e-10
        for k, v in gr.items():
            assert np.abs(v - g[k]).max() < 1e-10, k


def test_preproc_golden():
    """oracle.ops embed_nonseq / fuse_sequences / align_right vs the
    reference's embed_dense + embed_sparse + assemble_nonseq, fuse_sequences
    and align_right (preproc.py:103-152)."""
    from oracle import ops

    z = np.load(os.path.join(G, "preproc.npz"))
    p = {k[len("param:"):]: z[k] for k in z.files if k.startswith("param:")}
    g = {k[len("grad:"):]: z[k] for k in z.files if k.startswith("grad:")}
    fg = {k[len("fgrad:"):]: z[k] for k in z.files if k.startswith("fgrad:")}
    d, m, t_len = (int(v) for v in z["meta"][:3])
    vocabs = [int(v) for v in z["meta"][3:]]
    tabs = [p[f"emb/sparse{i}"] for i in range(len(vocabs))]
    out, bwd = ops.embed_nonseq(z["x"], z["ids"], p["emb/dense_proj"], tabs)
    assert np.abs(out - z["out"]).max() < 1e-12
    dproj, dts = bwd(z["cot"])
    assert np.abs(dproj - g["emb/dense_proj"]).max() < 1e-12
    for i, dt in enumerate(dts):
        assert np.abs(dt - g[f"emb/sparse{i}"]).max() < 1e-12
    al = ops.align_right([z["raw0"], z["raw1"]], t_len)
    assert np.array_equal(al[0], p["in/seq0"]) and np.array_equal(al[1], p["in/seq1"])
    ws, bs = [p["fus/w0"], p["fus/w1"]], [p["fus/b0"], p["fus/b1"]]
    fo, fb = ops.fuse_sequences(al, ws, bs, ["silu", "identity"])
    assert np.abs(fo - z["fused"]).max() < 1e-10
    dseqs, dws, dbs = fb(z["fcot"])
    for k in range(2):
        assert np.abs(dseqs[k] - fg[f"in/seq{k}"]).max() < 1e-10
    for i in range(2):
        assert np.abs(dws[i] - fg[f"fus/w{i}"]).max() < 1e-10
        assert np.abs(dbs[i] - fg[f"fus/b{i}"]).max() < 1e-10
