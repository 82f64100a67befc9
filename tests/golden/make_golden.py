"""Generate golden vectors by running the UNMODIFIED reference package.

Run in the build container (the only place /root/reference exists):

    python tests/golden/make_golden.py

It imports ``kunlun`` from /root/reference/pkg/src, evaluates each hot-path
op (and a composed 2-layer model following SURVEY.md Appendix A.1, since the
reference ships no model module) under the reference's own Tape, and writes
inputs, parameters, outputs and gradients to ``tests/golden/*.npz``.  The
committed fixtures pin both the numpy oracle (tests/test_oracle_golden.py)
and, through the oracle, the CUDA kernels.

Oracle workarounds: the scalar loss is reshaped to 0-d
before ``backward`` (tensor.py:36 vs 200-201), and inputs are registered as
Params to obtain their gradients (tensor.py:219-224).
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
# the repo root first (for ``oracle``), then the reference in front of it, so
# ``import kunlun`` resolves to the unmodified reference, not the repo's
# B200 drop-in package of the same name
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, REF)
# the reference's kunlun is a namespace package: a regular package of the same
# name anywhere on sys.path (the repo's B200 drop-in kunlun/) would win, so
# bind the name to the reference's directory explicitly
import types  # noqa: E402

_ref_pkg = types.ModuleType("kunlun")
_ref_pkg.__path__ = [os.path.join(REF, "kunlun")]
sys.modules["kunlun"] = _ref_pkg

from kunlun import attention as A  # noqa: E402
from kunlun import gdpa as G  # noqa: E402
from kunlun import interaction as I  # noqa: E402
from kunlun import mlp as M  # noqa: E402
from kunlun import preproc as PP  # noqa: E402
from kunlun import seqsum as Q  # noqa: E402
from kunlun import tensor as T  # noqa: E402

from oracle import model as OM  # noqa: E402  (only for the shared init / spec)


def _backward(tape, loss):
    # sum_all's VJP broadcasts the 0-d seed back to the (1,)-shaped scalars
    # the reference produces (tensor.py:36 promotion), then reshape to 0-d.
    with tape:
        loss = T.sum_all(loss)
    loss.data = loss.data.reshape(())
    return T.backward(tape, loss)


def _dot(out, r):
    return T.sum_all(T.mul(out, T.constant(r)))


def _save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print("wrote", path, sum(a.size for a in arrays.values()), "values")


def _mha_params(params, prefix):
    H = 0
    while f"{prefix}/head{H}/w_q" in params:
        H += 1
    return A.MhaParams([params[f"{prefix}/head{h}/w_q"] for h in range(H)],
                       [params[f"{prefix}/head{h}/w_k"] for h in range(H)],
                       [params[f"{prefix}/head{h}/w_v"] for h in range(H)],
                       params[f"{prefix}/w_out"])


def _wg_params(params, prefix):
    H = 0
    while f"{prefix}/head{H}/w_q" in params:
        H += 1
    return G.WeightGenParams([params[f"{prefix}/head{h}/w_q"] for h in range(H)],
                             [params[f"{prefix}/head{h}/w_kgen"] for h in range(H)],
                             [params[f"{prefix}/head{h}/w_vgen"] for h in range(H)],
                             params[f"{prefix}/w_out"])


def _summ_params(params, prefix, budget):
    split = Q.SummarySplit.for_budget(budget)
    rank = 0
    while f"{prefix}/hsp/kron{rank}/seq_map" in params:
        rank += 1
    hsp = Q.HspParams(params[f"{prefix}/hsp/seeds"], params[f"{prefix}/hsp/norm_gain"],
                      _mha_params(params, f"{prefix}/hsp/attn"),
                      [params[f"{prefix}/hsp/kron{i}/seq_map"] for i in range(rank)],
                      [params[f"{prefix}/hsp/kron{i}/emb_map"] for i in range(rank)])
    if split.n_cls > 0:
        return Q.SummarizerParams(hsp, params[f"{prefix}/cls_queries"],
                                  _mha_params(params, f"{prefix}/cls_attn"), split)
    return Q.SummarizerParams(hsp, None, None, split)


def _gi_params(params, prefix, total, experts, d):
    part = I.ExpertPartition.contiguous(total, experts)
    exps = []
    for i in range(experts):
        deep = M.Mlp([params[f"{prefix}/expert{i}/deep/w0"], params[f"{prefix}/expert{i}/deep/w1"]],
                     [params[f"{prefix}/expert{i}/deep/b0"], params[f"{prefix}/expert{i}/deep/b1"]],
                     ["silu", "identity"])
        exps.append(I.WukongExpertParams(params[f"{prefix}/expert{i}/dot_map"], deep,
                                         params[f"{prefix}/expert{i}/gate_dot"],
                                         params[f"{prefix}/expert{i}/gate_deep"]))
    return I.InteractionParams(exps, part, params[f"{prefix}/aggregate"])


def _registry(pdict):
    params = T.Params()
    for k, v in pdict.items():
        params.add(k, v)
    return params


def _pack(prefix, d):
    return {f"{prefix}:{k}": np.asarray(v, dtype=np.float64) for k, v in d.items()}


# ---------------------------------------------------------------------------


def case_gdpa(rng, acts, tag, wscale=1.0):
    """gdpa.summarize_nonseq + generate_kv + gdpa_forward_blockwise."""
    d, H, n_kv, n_sum, n_ctx, t_len = 16, 4, 4, 2, 5, 12
    cfg = G.GdpaConfig(dim=d, heads=H, n_kv=n_kv, tau=float(t_len), activations=tuple(acts))
    params = T.Params()
    wg = G.WeightGenParams.create(params, "g", cfg, n_sum, d, rng)
    for name, t in params.items():
        t.data = t.data * wscale
    pool = params.add("pool", rng.normal(0, 1 / np.sqrt(n_ctx), (n_sum, n_ctx)))
    s = params.add("in/S", rng.normal(0, 1 / np.sqrt(d), (t_len, d)))
    x = params.add("in/X", rng.normal(0, 1, (n_ctx, d)))
    r = rng.normal(0, 1, (t_len, d))
    with T.Tape(params) as tape:
        xs = G.summarize_nonseq(x, pool)
        y = G.gdpa_forward_blockwise(s, xs, cfg, wg, block_t=5, block_kv=3)
        loss = _dot(y, r)
    grads = _backward(tape, loss)
    yref = G.gdpa_forward(Tensor_(s), G.summarize_nonseq(Tensor_(x), Tensor_(pool)), cfg, wg).data
    assert np.abs(yref - y.data).max() < 1e-10
    _save(f"gdpa_{tag}.npz", acts=np.array(acts), **_pack("param", {k: v.data for k, v in params.items()}),
          **_pack("grad", {k: v.data for k, v in grads.items()}), out_Y=y.data, cot_Y=r,
          meta=np.array([d, H, n_kv, n_sum, n_ctx, t_len]))


def Tensor_(t):
    return T.Tensor(t.data)


def case_mha(rng, t_len, w, causal, length, tag, full=False):
    d, H = 16, 2
    params = T.Params()
    mp = A.MhaParams.create(params, "m", d, H, rng)
    s = params.add("in/S", rng.normal(0, 1, (t_len, d)))
    r = rng.normal(0, 1, (t_len, d))
    with T.Tape(params) as tape:
        if full:
            y = A.mha_full(s, mp, length=length)
        else:
            y = A.mha_window(s, mp, A.WindowSpec(w, causal), length=length)
        loss = _dot(y, r)
    grads = _backward(tape, loss)
    _save(f"mha_{tag}.npz", **_pack("param", {k: v.data for k, v in params.items()}),
          **_pack("grad", {k: v.data for k, v in grads.items()}), out_Y=y.data, cot_Y=r,
          meta=np.array([d, H, t_len, w, int(causal), -1 if length is None else length, int(full)]))


def case_hsp(rng, t_len, tag):
    d, H, budget, n_seeds, rank = 16, 2, 8, 6, 2
    params = T.Params()
    sp = Q.SummarizerParams.create(params, "s", d, Q.SummarySplit.for_budget(budget), n_seeds, rank, H, rng)
    s = params.add("in/S", rng.normal(0, 1, (t_len, d)))
    with T.Tape(params) as tape:
        bundle = Q.hsp_summarize(s, sp)
        rows = bundle.rows()
        r = rng.normal(0, 1, rows.shape)
        loss = _dot(rows, r)
    grads = _backward(tape, loss)
    _save(f"hsp_{tag}.npz", **_pack("param", {k: v.data for k, v in params.items()}),
          **_pack("grad", {k: v.data for k, v in grads.items()}), out_Y=rows.data, cot_Y=r,
          meta=np.array([d, H, t_len, budget, n_seeds, rank]))


def case_gi(rng):
    d, n_ctx, experts, hidden = 8, 5, 2, 16
    budgets = [8, 4]
    total = n_ctx + sum(budgets)
    params = T.Params()
    part = I.ExpertPartition.contiguous(total, experts)
    ip = I.InteractionParams.create(params, "gi", part, n_ctx, d, hidden, rng)
    x = params.add("in/X", rng.normal(0, 1, (n_ctx, d)))
    rows = [params.add(f"in/R{e}", rng.normal(0, 1, (b, d))) for e, b in enumerate(budgets)]
    r = rng.normal(0, 1, (n_ctx, d))
    with T.Tape(params) as tape:
        y = I.global_interaction(x, rows, ip)
        loss = _dot(y, r)
    grads = _backward(tape, loss)
    _save("gi.npz", **_pack("param", {k: v.data for k, v in params.items()}),
          **_pack("grad", {k: v.data for k, v in grads.items()}), out_Y=y.data, cot_Y=r,
          meta=np.array([d, n_ctx, experts, hidden] + budgets))


def case_model(rng, compskip, tag):
    """2-layer, 2-event composed model per SURVEY.md Appendix A.1, evaluated
    with the reference modules and Tape; loss = BCE + sum_l <out_l, R_l>."""
    spec = OM.ModelSpec(L=2, d=16, heads=4, n_ctx=5, n_sum=2, n_kv=4, experts=2, compskip=compskip,
                        events=[OM.EventSpec(T=12, w=3, budget=8, n_seeds=6, rank=2),
                                OM.EventSpec(T=9, w=2, budget=4, n_seeds=3, rank=1)])
    pdict = OM.init_params(spec, seed=int(rng.integers(1 << 30)))
    B = 3
    lengths = [np.array([12, 5, 0]), np.array([9, 1, 9])]
    X = rng.normal(0, 1 / np.sqrt(spec.d), (B, spec.n_ctx, spec.d))
    S = [rng.normal(0, 1 / np.sqrt(spec.d), (B, ev.T, spec.d)) for ev in spec.events]
    labels = (rng.random(B) < 0.3).astype(np.float64)
    cot = [{"X": rng.normal(0, 0.1, X.shape),
            "S": [rng.normal(0, 0.1, s.shape) for s in S],
            "H": [rng.normal(0, 0.1, (B, ev.budget, spec.d)) for ev in spec.events]} for _ in range(spec.L)]
    params = _registry(pdict)
    flags = OM.compskip_config(spec.L, compskip)
    n_tot = spec.n_tot
    logits = []
    extra = []
    with T.Tape(params) as tape:
        for b in range(B):
            x = params.add(f"in/X{b}", X[b])
            s_list = [params.add(f"in/S{e}_{b}", S[e][b, : lengths[e][b]]) for e in range(2)]
            H = None
            for l in range(spec.L):
                skip_attn, skip_hsp, skip_pffn = flags[l]
                xsum = G.summarize_nonseq(x, params[f"L{l}/pool"])
                Hn = []
                for e, ev in enumerate(spec.events):
                    if skip_hsp:
                        Hn.append(H[e])
                    else:
                        Hn.append(Q.hsp_summarize(s_list[e], _summ_params(params, f"L{l}/ev{e}/summ", ev.budget)).rows())
                xn = I.global_interaction(x, Hn, _gi_params(params, f"L{l}/gi", n_tot, spec.experts, spec.d))
                sn = []
                for e, ev in enumerate(spec.events):
                    st = s_list[e]
                    cfg = G.GdpaConfig(dim=spec.d, heads=spec.heads, n_kv=spec.n_kv, tau=float(ev.T))
                    if not skip_pffn:
                        wg = _wg_params(params, f"L{l}/ev{e}/gdpa")
                        kv = G.generate_kv(xsum, wg, cfg)
                        st = G.gdpa_forward_blockwise(st, xsum, cfg, wg, kv=kv)
                    if not skip_attn:
                        st = A.mha_window(st, _mha_params(params, f"L{l}/ev{e}/mha"), A.WindowSpec(ev.w))
                    sn.append(st)
                x, s_list, H = xn, sn, Hn
                extra.append(_dot(x, cot[l]["X"][b]))
                for e in range(2):
                    extra.append(_dot(s_list[e], cot[l]["S"][e][b, : lengths[e][b]]))
                    extra.append(_dot(H[e], cot[l]["H"][e][b]))
            head = M.Mlp([params["head/w0"], params["head/w1"]], [params["head/b0"], params["head/b1"]],
                         ["silu", "identity"])
            logits.append(head.apply_vec(T.reshape(x, (spec.n_ctx * spec.d,))))
        z = T.concat(logits, axis=0)
        loss = T.bce_with_logits(z, labels)
        for t in extra:
            loss = T.add(loss, t)
    grads = _backward(tape, loss)
    dX = np.stack([grads[f"in/X{b}"].data for b in range(B)])
    dS = [np.zeros_like(s) for s in S]
    for e in range(2):
        for b in range(B):
            dS[e][b, : lengths[e][b]] = grads[f"in/S{e}_{b}"].data
            dS[e][b, lengths[e][b]:] = sum(cot[l]["S"][e][b, lengths[e][b]:] for l in range(spec.L))
    arrays = {"X": X, "labels": labels, "loss": np.asarray(loss.data, dtype=np.float64).reshape(()), "logits": z.data, "dX": dX}
    for e in range(2):
        arrays[f"S{e}"] = S[e]
        arrays[f"len{e}"] = lengths[e]
        arrays[f"dS{e}"] = dS[e]
    for l in range(spec.L):
        arrays[f"cot{l}_X"] = cot[l]["X"]
        for e in range(2):
            arrays[f"cot{l}_S{e}"] = cot[l]["S"][e]
            arrays[f"cot{l}_H{e}"] = cot[l]["H"][e]
    arrays.update(_pack("param", pdict))
    arrays.update(_pack("grad", {k: v.data for k, v in grads.items() if not k.startswith("in/")}))
    _save(f"model_{tag}.npz", **arrays)


def case_index():
    """Integer/bool KATs straight from the reference (bit-exact targets)."""
    arrays = {}
    for t_len in (1, 2, 6, 13, 130, 257):
        for w in (0, 1, 5, 64, 128):
            for causal in (False, True):
                arrays[f"band_{t_len}_{w}_{int(causal)}"] = A.band_mask(t_len, w, causal)
                arrays[f"support_{t_len}_{w}_{int(causal)}"] = A.band_support_sizes(t_len, w, causal)
    for total in (3, 13, 41, 48, 97):
        for m in (1, 2, 3, 5):
            if m <= total:
                arrays[f"experts_{total}_{m}"] = np.array(I.ExpertPartition.contiguous(total, m).ranges)
    for budget in (1, 4, 8, 13, 32, 64):
        s = Q.SummarySplit.for_budget(budget)
        arrays[f"split_{budget}"] = np.array([s.n_cls, s.n_tokens, s.n_recent])
    class _ZeroRng:
        """Noise-free generator: exposes the exact seed->token init pattern."""

        def normal(self, loc, scale, size):
            return np.zeros(size)

    for n_s, n_t in ((8, 4), (32, 16), (6, 4), (7, 3), (64, 16), (5, 4)):
        params = T.Params()
        hp = Q.HspParams.create(params, "h", 4, n_s, n_t, 1, 1, _ZeroRng())
        arrays[f"hspbase_{n_s}_{n_t}"] = hp.seq_maps[0].data
    for t_len in (0, 1, 3, 8):
        s = T.Tensor(np.arange(t_len * 2, dtype=np.float64).reshape(t_len, 2))
        arrays[f"recent_{t_len}"] = Q.recent_rows(s, 4).data
    arrays["attention_macs"] = np.array([A.attention_macs(256, 64, 28864), A.attention_macs(1024, 256, 246656)])
    _save("index.npz", **arrays)


def case_rote():
    """ROTE (preproc.py:155-199, tensor.py:508-532): rote_sequence on (T, d)
    rows with and without timestamps, both gap modes, default and custom
    frequency schedules; output and input gradient under a random cotangent."""
    rng = np.random.default_rng(20261019)
    out = {}
    cases = [("prev", 8, 7, "previous", True, None), ("latest", 8, 7, "latest", True, None),
             ("nots", 6, 5, "previous", False, None), ("custom", 4, 9, "latest", True, 17.0),
             ("empty", 4, 0, "previous", True, None)]
    for tag, d, t_len, mode, with_ts, tau_scale in cases:
        if tau_scale is None:
            cfg = PP.RoteConfig.default(d, gap_mode=mode)
        else:
            cfg = PP.RoteConfig(rng.uniform(0.01, 2.0, d // 2), rng.uniform(0.01, 2.0, d // 2), tau_scale, mode)
        params = T.Params()
        s = params.add("in/S", rng.normal(0, 1, (t_len, d)))
        ts = np.cumsum(rng.exponential(120.0, t_len)) if with_ts else None
        r = rng.normal(0, 1, (t_len, d))
        with T.Tape(params) as tape:
            y = PP.rote_sequence(s, ts, cfg)
            loss = _dot(y, r)
        if t_len:
            g = _backward(tape, loss)["in/S"].data
        else:
            g = np.zeros((0, d))
        out.update({f"{tag}:S": s.data, f"{tag}:ts": np.zeros(0) if ts is None else ts, f"{tag}:has_ts": np.array(int(with_ts)),
                    f"{tag}:pos": cfg.pos_freqs, f"{tag}:temp": cfg.temp_freqs, f"{tag}:tau_scale": np.array(cfg.tau_scale),
                    f"{tag}:mode": np.array(0 if mode == "previous" else 1), f"{tag}:Y": y.data, f"{tag}:cot": r,
                    f"{tag}:dS": g})
    _save("rote.npz", **out)


def case_ablation():
    """Table 2 ablation baselines from the reference's own building blocks:
    gdpa.pffn_original (gdpa.py:227-257) and a PMA-only summary
    [CLS | pma(Q_learn, S) | recent] (seqsum.py:26-34, 186-196)."""
    rng = np.random.default_rng(20261019)
    d, n_sum, n_ctx, t_len, hidden = 8, 2, 5, 9, 12
    params = T.Params()
    pp = G.PffnParams.create(params, "pf", d, n_sum, d, hidden, rng)
    s = params.add("in/S", rng.normal(0, 1 / np.sqrt(d), (t_len, d)))
    xsum = params.add("in/Xsum", rng.normal(0, 1, (n_sum, d)))
    r = rng.normal(0, 1, (t_len, d))
    with T.Tape(params) as tape:
        y = G.pffn_original(xsum, s, pp)
        loss = _dot(y, r)
    grads = _backward(tape, loss)
    _save("pffn_original.npz", **_pack("param", {k: v.data for k, v in params.items()}),
          **_pack("grad", {k: v.data for k, v in grads.items()}), out_Y=y.data, cot_Y=r,
          meta=np.array([d, n_sum, n_ctx, t_len, hidden]))
    for t_len, tag in ((10, "t10"), (0, "t0")):
        d, H, budget = 16, 2, 8
        n_cls, n_tok, n_rec = 2, 4, 2
        params = T.Params()
        cq = params.add("s/cls_queries", rng.normal(0, 1 / np.sqrt(d), (n_cls, d)))
        ca = A.MhaParams.create(params, "s/cls_attn", d, H, rng)
        pq = params.add("s/pma_queries", rng.normal(0, 1 / np.sqrt(d), (n_tok, d)))
        pa = A.MhaParams.create(params, "s/pma_attn", d, H, rng)
        s = params.add("in/S", rng.normal(0, 1, (t_len, d)))
        r = rng.normal(0, 1, (budget, d))
        with T.Tape(params) as tape:
            if t_len:
                rows = T.concat([Q.pma(s, cq, ca), Q.pma(s, pq, pa), Q.recent_rows(s, n_rec)], axis=0)
            else:
                rows = T.constant(np.zeros((budget, d)))
            loss = _dot(rows, r)
        grads = _backward(tape, loss) if t_len else {k: T.Tensor(np.zeros_like(v.data)) for k, v in params.items()}
        _save(f"pma_summary_{tag}.npz", **_pack("param", {k: v.data for k, v in params.items()}),
              **_pack("grad", {k: v.data for k, v in grads.items()}), out_rows=rows.data, cot=r,
              meta=np.array([d, H, budget, t_len]))


def case_preproc():
    """preproc.embed_dense / embed_sparse / assemble_nonseq / fuse_sequences /
    align_right of the reference (preproc.py:103-152)."""
    rng = np.random.default_rng(20261020)
    d, m, vocabs = 8, 3, [5, 7, 2]
    params = T.Params()
    proj = params.add("emb/dense_proj", rng.normal(0, 1 / np.sqrt(m), (d, m)))
    tabs = [params.add(f"emb/sparse{i}", rng.normal(0, 1 / np.sqrt(d), (v, d))) for i, v in enumerate(vocabs)]
    x = rng.normal(0, 1, m)
    ids = np.array([4, 0, 1])
    r = rng.normal(0, 1, (len(vocabs) + 1, d))
    with T.Tape(params) as tape:
        out = PP.assemble_nonseq(PP.embed_dense(x, proj), [PP.embed_sparse(i, t) for i, t in zip(ids, tabs)])
        loss = _dot(out, r)
    grads = _backward(tape, loss)
    # fusion of K = 2 right-aligned sequences
    K_, t_len = 2, 6
    fusion = M.Mlp.create(params, "fus", [K_ * d, 12, d], ["silu", "identity"], rng)
    raw = [rng.normal(0, 1, (4, d)), rng.normal(0, 1, (6, d))]
    al = PP.align_right(raw, t_len)
    seqs = [params.add(f"in/seq{k}", a) for k, a in enumerate(al)]
    rf = rng.normal(0, 1, (t_len, d))
    with T.Tape(params) as tape:
        fo = PP.fuse_sequences(seqs, fusion)
        loss = _dot(fo, rf)
    fgrads = _backward(tape, loss)
    _save("preproc.npz", **_pack("param", {k: v.data for k, v in params.items()}),
          **_pack("grad", {k: v.data for k, v in grads.items()}),
          **_pack("fgrad", {k: v.data for k, v in fgrads.items()}),
          x=x, ids=ids, out=out.data, cot=r, fused=fo.data, fcot=rf, raw0=raw[0], raw1=raw[1],
          meta=np.array([d, m, t_len] + vocabs))


def main():
    rng = np.random.default_rng(20260218)
    case_gdpa(rng, ("silu", "relu", "identity", "tanh"), "default")
    case_gdpa(rng, ("sigmoid", "exp", "silu", "relu"), "sigexp", wscale=0.5)
    case_mha(rng, 13, 3, False, 9, "w3_len9")
    case_mha(rng, 13, 3, True, None, "w3_causal")
    case_mha(rng, 11, 20, False, 7, "full_len7", full=True)
    case_mha(rng, 6, 0, False, 0, "w0_len0")
    case_hsp(rng, 10, "t10")
    case_hsp(rng, 1, "t1")
    case_hsp(rng, 0, "t0")
    case_gi(rng)
    case_model(rng, False, "noskip")
    case_model(rng, True, "compskip")
    case_index()


if __name__ == "__main__":
    if sys.argv[1:] == ["rote"]:
        case_rote()
    elif sys.argv[1:] == ["ablation"]:
        case_ablation()
    elif sys.argv[1:] == ["preproc"]:
        case_preproc()
    else:
        main()
        case_rote()
        case_ablation()
        case_preproc()
