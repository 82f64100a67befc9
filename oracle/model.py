"""Kunlun layer / model composition (oracle; test infrastructure only).

The reference ships no ``model`` module; the composition is
restated from SPEC.md:474-533 and PAPER.md:515-541 (Alg. 1) / 586-603
(Alg. 4) exactly as SURVEY.md Appendix A.1 pins it, on top of the per-module
restatements in ``oracle.kunlun``.  Sequences are handled per sample on their
valid rows only (jagged semantics, jagged.py:10-100); padding rows pass
through every layer unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import kunlun as K
from .ops import bce_with_logits, mlp_rows

DEFAULT_ACTIVATION_CYCLE = K.DEFAULT_ACTIVATION_CYCLE


@dataclass
class EventSpec:
    T: int
    w: int
    budget: int
    n_seeds: int
    rank: int
    causal: bool = False
    d: int = 0        # event width / heads / depth (0 = the model's): event-level
    heads: int = 0    # personalization
    layers: int = 0


@dataclass
class ModelSpec:
    L: int
    d: int
    heads: int
    n_ctx: int                 # n + 1 non-sequence tokens
    events: list
    n_sum: int = 4
    n_kv: int = 16
    experts: int = 2
    compskip: bool = False
    gdpa_acts: tuple = ()
    expert_hidden: int = 0     # default 2d
    head_hidden: int = 0       # default 4d
    pffn: str = "gdpa"         # Table 2 ablations: "original" (gdpa.py:227-257)
    summarizer: str = "hsp"    # "pma": learnable-query PMA summaries
    attention: str = "window"  # "full": mha_full (attention.py:115-121)
    pffn_hidden: int = 0       # default 2d

    def __post_init__(self):
        if not self.gdpa_acts:
            c = DEFAULT_ACTIVATION_CYCLE
            self.gdpa_acts = tuple(c[h % len(c)] for h in range(self.heads))
        if not self.expert_hidden:
            self.expert_hidden = 2 * self.d
        if not self.head_hidden:
            self.head_hidden = 4 * self.d
        if not self.pffn_hidden:
            self.pffn_hidden = 2 * self.d

    @property
    def n_tot(self) -> int:
        return self.n_ctx + sum(e.budget for e in self.events)

    def ev_d(self, e: int) -> int:
        return self.events[e].d or self.d

    def ev_heads(self, e: int) -> int:
        return self.events[e].heads or self.heads

    def ev_layers(self, e: int) -> int:
        return self.events[e].layers or self.L

    def ev_acts(self, e: int) -> tuple:
        H = self.ev_heads(e)
        if H == self.heads:
            return tuple(self.gdpa_acts)
        return tuple(DEFAULT_ACTIVATION_CYCLE[h % len(DEFAULT_ACTIVATION_CYCLE)] for h in range(H))


def compskip_config(L: int, enabled: bool = True):
    """Alg. 4: even l -> (skip_attn=T,
    skip_hsp=F, skip_pffn=F); odd l -> (F, T, T); disabled -> all F."""
    if L < 1:
        raise ValueError("need at least one layer")
    if not enabled:
        return [(False, False, False) for _ in range(L)]
    return [(True, False, False) if l % 2 == 0 else (False, True, True) for l in range(L)]


def init_params(spec: ModelSpec, seed: int = 0) -> dict:
    """Registry-named float64 parameters with the reference initializers'
    distributions (gdpa.py:83-93, attention.py:33-46, seqsum.py:58-77 and
    177-183, interaction.py:87-99/133-141, mlp.py:26-34)."""
    rng = np.random.default_rng(seed)
    d, H = spec.d, spec.heads
    d_h = d // H
    p = {}

    def mha(prefix, dd=d, HH=H):
        sig = 1.0 / np.sqrt(dd)
        for h in range(HH):
            p[f"{prefix}/head{h}/w_q"] = rng.normal(0.0, sig, (dd // HH, dd))
            p[f"{prefix}/head{h}/w_k"] = rng.normal(0.0, sig, (dd // HH, dd))
            p[f"{prefix}/head{h}/w_v"] = rng.normal(0.0, sig, (dd // HH, dd))
        p[f"{prefix}/w_out"] = rng.normal(0.0, 0.5 * sig, (dd, dd))

    def mlp(prefix, widths):
        for i, (fi, fo) in enumerate(zip(widths[:-1], widths[1:])):
            p[f"{prefix}/w{i}"] = rng.normal(0.0, 1.0 / np.sqrt(fi), (fo, fi))
            p[f"{prefix}/b{i}"] = np.zeros(fo)

    ranges = K.expert_ranges(spec.n_tot, spec.experts)
    for l in range(spec.L):
        p[f"L{l}/pool"] = rng.normal(0.0, 1.0 / np.sqrt(spec.n_ctx), (spec.n_sum, spec.n_ctx))
        for e, ev in enumerate(spec.events):
            if l >= spec.ev_layers(e):  # the event's stack ended (hold-last)
                continue
            dd, HH = spec.ev_d(e), spec.ev_heads(e)
            dh = dd // HH
            fan = spec.n_sum * d
            if spec.pffn == "original":  # gdpa.py:235-245
                pre = f"L{l}/ev{e}/pffn"
                hid = spec.pffn_hidden
                p[f"{pre}/w1"] = rng.normal(0.0, 1.0 / np.sqrt(fan), (hid, fan))
                p[f"{pre}/b1"] = np.zeros(hid)
                p[f"{pre}/w2"] = rng.normal(0.0, 0.1 / np.sqrt(hid), (dd * dd, hid))
                p[f"{pre}/b2"] = np.zeros(dd * dd)
            else:
                pre = f"L{l}/ev{e}/gdpa"
                for h in range(HH):
                    p[f"{pre}/head{h}/w_q"] = rng.normal(0.0, 1.0 / np.sqrt(dd), (dh, dd))
                    p[f"{pre}/head{h}/w_kgen"] = rng.normal(0.0, 1.0 / np.sqrt(fan), (spec.n_kv * dh, fan))
                    p[f"{pre}/head{h}/w_vgen"] = rng.normal(0.0, 1.0 / np.sqrt(fan), (spec.n_kv * dh, fan))
                p[f"{pre}/w_out"] = rng.normal(0.0, 0.5 / np.sqrt(dd), (dd, dd))
            mha(f"L{l}/ev{e}/mha", dd, HH)
            if dd != d:  # learnable linear adapter of the summaries
                p[f"L{l}/ev{e}/adapter"] = rng.normal(0.0, 1.0 / np.sqrt(dd), (d, dd))
            n_cls, n_tok, _ = K.split_for_budget(ev.budget)
            sp = f"L{l}/ev{e}/summ"
            if spec.summarizer == "pma":
                if n_cls > 0:
                    p[f"{sp}/cls_queries"] = rng.normal(0.0, 1.0 / np.sqrt(dd), (n_cls, dd))
                    mha(f"{sp}/cls_attn", dd, HH)
                p[f"{sp}/pma_queries"] = rng.normal(0.0, 1.0 / np.sqrt(dd), (n_tok, dd))
                mha(f"{sp}/pma_attn", dd, HH)
                continue
            p[f"{sp}/hsp/seeds"] = rng.normal(0.0, 1.0 / np.sqrt(dd), (ev.n_seeds, dd))
            p[f"{sp}/hsp/norm_gain"] = np.ones(dd)
            mha(f"{sp}/hsp/attn", dd, HH)
            base = np.zeros((ev.n_seeds, n_tok))
            bounds = K.hsp_init_bounds(ev.n_seeds, n_tok)
            for j in range(n_tok):
                lo, hi = bounds[j], max(bounds[j + 1], bounds[j] + 1)
                base[lo:hi, j] = 1.0 / (hi - lo)
            for i in range(ev.rank):
                p[f"{sp}/hsp/kron{i}/seq_map"] = base / ev.rank + rng.normal(0.0, 0.02, (ev.n_seeds, n_tok))
                p[f"{sp}/hsp/kron{i}/emb_map"] = np.eye(dd) + rng.normal(0.0, 0.02, (dd, dd))
            if n_cls > 0:
                p[f"{sp}/cls_queries"] = rng.normal(0.0, 1.0 / np.sqrt(dd), (n_cls, dd))
                mha(f"{sp}/cls_attn", dd, HH)
        gp = f"L{l}/gi"
        for i, (a, b) in enumerate(ranges):
            n_i = b - a
            n_pairs = n_i * (n_i + 1) // 2
            p[f"{gp}/expert{i}/dot_map"] = rng.normal(0.0, 0.1 / np.sqrt(n_pairs), (n_i * d, n_pairs))
            mlp(f"{gp}/expert{i}/deep", [d, spec.expert_hidden, d])
            p[f"{gp}/expert{i}/gate_dot"] = np.ones(1)
            p[f"{gp}/expert{i}/gate_deep"] = np.ones(1)
        p[f"{gp}/aggregate"] = rng.normal(0.0, 0.1 / np.sqrt(spec.n_tot), (spec.n_ctx, spec.n_tot))
    mlp("head", [spec.n_ctx * d, spec.head_hidden, 1])
    return p


def layer_forward(spec: ModelSpec, p: dict, l: int, flags, X, S_list, H_prev):
    """One Kunlun layer on one sample (Alg. 1).

    ``S_list[e]`` holds only the valid rows of event e.  Returns
    (X', S'_list, H_list, bwd) where bwd(dX', dS'_list, dH_list) returns
    (dX, dS_list, dH_prev_list, grads)."""
    skip_attn, skip_hsp, skip_pffn = flags
    if skip_hsp and H_prev is None:
        raise ValueError("skip_hsp on a layer without H_prev")
    xsum, xs_bwd = K.summarize_nonseq(X, p[f"L{l}/pool"])
    kv, kv_bwd = [], []
    H_list, h_bwd = [], []
    ended = [l >= spec.ev_layers(e) for e in range(len(spec.events))]  # hold-last events
    for e, ev in enumerate(spec.events):
        if skip_pffn or spec.pffn == "original" or ended[e]:
            kv.append(None)
            kv_bwd.append(None)
        else:
            a, b = K.generate_kv(xsum, p, f"L{l}/ev{e}/gdpa", spec.n_kv)
            kv.append(a)
            kv_bwd.append(b)
        if skip_hsp or ended[e]:
            H_list.append(H_prev[e])
            h_bwd.append(None)
        else:
            summ = K.pma_summarize if spec.summarizer == "pma" else K.hsp_summarize
            rows, rb = summ(S_list[e], p, f"L{l}/ev{e}/summ", ev.budget)
            akey = f"L{l}/ev{e}/adapter"
            if akey in p:  # d_e -> d linear adapter
                A = p[akey]
                rows_e = rows
                rows = rows_e @ A.T

                def rb(g, rb=rb, rows_e=rows_e, A=A, akey=akey):
                    ds, gr = rb(g @ A)
                    K._acc(gr, akey, g.T @ rows_e)
                    return ds, gr
            H_list.append(rows)
            h_bwd.append(rb)
    Xn, gi_bwd = K.global_interaction(X, H_list, p, f"L{l}/gi", spec.experts)
    S_out, s_bwd = [], []
    for e, ev in enumerate(spec.events):
        s = S_list[e]
        if ended[e]:  # the event's sequence passes through
            S_out.append(s)
            s_bwd.append((None, None))
            continue
        if skip_pffn:
            st, gb = s, None
        elif spec.pffn == "original":
            st, pb = K.pffn_original(xsum, s, p, f"L{l}/ev{e}/pffn")
            gb = ("original", pb)
        else:
            st, gb = K.gdpa_forward(s, kv[e], p, f"L{l}/ev{e}/gdpa", float(ev.T), spec.ev_acts(e))
        if skip_attn:
            so, ab = st, None
        elif spec.attention == "full":
            so, ab = K.mha_full(st, p, f"L{l}/ev{e}/mha")
        else:
            so, ab = K.mha_window(st, p, f"L{l}/ev{e}/mha", ev.w, ev.causal)
        S_out.append(so)
        s_bwd.append((gb, ab))

    def bwd(dXn, dS_list, dH_list):
        grads = {}
        dX, dHrows, gr = gi_bwd(dXn)
        K.merge_grads(grads, gr)
        dS_in, dH_prev = [], []
        dxsum = np.zeros_like(xsum)
        for e in range(len(spec.events)):
            gb, ab = s_bwd[e]
            g = dS_list[e]
            if ab is not None:
                g, gr = ab(g)
                K.merge_grads(grads, gr)
            if isinstance(gb, tuple):  # pffn_original: dS and dX_sum directly
                g, dxs, gr = gb[1](g)
                K.merge_grads(grads, gr)
                dxsum = dxsum + dxs
            elif gb is not None:
                g, dkvs, gr = gb(g)
                K.merge_grads(grads, gr)
                dxs, gr = kv_bwd[e](dkvs)
                K.merge_grads(grads, gr)
                dxsum = dxsum + dxs
            dH = dHrows[e] + (dH_list[e] if dH_list is not None and dH_list[e] is not None else 0.0)
            if h_bwd[e] is None:
                dH_prev.append(dH)
            else:
                ds_h, gr = h_bwd[e](dH)
                K.merge_grads(grads, gr)
                g = g + ds_h
                dH_prev.append(None)
            dS_in.append(g)
        dX_s, dpool = xs_bwd(dxsum)
        grads[f"L{l}/pool"] = dpool
        return dX + dX_s, dS_in, dH_prev, grads

    return Xn, S_out, H_list, bwd


def model_forward_backward(spec: ModelSpec, p: dict, X, S, lengths, labels, cot=None):
    """Full model on a padded batch: X (B, n_ctx, d), S[e] (B, T_e, d),
    lengths[e] (B,), labels (B,).  Loss = mean BCE(head(flatten X^(L)))
    (tensor.py:535-549; head Mlp [(n+1)d, 4d, 1] silu/identity)
    plus, if ``cot`` is given, sum_l <out_l, R_l> over every layer output
    (SURVEY.md §4.2 L3 parity loss).  ``cot[l] = {"X": (B,n_ctx,d),
    "S": [ (B,T_e,d) ], "H": [ (B,budget_e,d) ]}``.

    Returns dict(loss, logits, outs, grads, dX, dS) — dS/outs in the padded
    layout (pad rows pass through: their output equals the input)."""
    B = X.shape[0]
    flags = compskip_config(spec.L, spec.compskip)
    logits = np.zeros(B)
    grads: dict = {}
    dX_all = np.zeros_like(X)
    dS_all = [np.zeros_like(s) for s in S]
    outs = [{"X": np.zeros_like(X), "S": [np.zeros_like(s) for s in S],
             "H": [np.zeros((B, ev.budget, spec.d)) for ev in spec.events]} for _ in range(spec.L)]
    hw = [p["head/w0"], p["head/w1"]]
    hb = [p["head/b0"], p["head/b1"]]
    per_sample = []
    for b in range(B):
        x = X[b]
        s_list = [S[e][b, : lengths[e][b]] for e in range(len(spec.events))]
        H = None
        bwds = []
        for l in range(spec.L):
            x, s_list, H, bw = layer_forward(spec, p, l, flags[l], x, s_list, H)
            bwds.append(bw)
            outs[l]["X"][b] = x
            for e in range(len(spec.events)):
                full = S[e][b].copy()
                full[: lengths[e][b]] = s_list[e]
                outs[l]["S"][e][b] = full
                outs[l]["H"][e][b] = H[e]
        flat = x.reshape(-1)
        z, h_bwd = mlp_rows(flat[None, :], hw, hb, ["silu", "identity"])
        logits[b] = z[0, 0]
        per_sample.append((bwds, h_bwd))
    loss, bce_bwd = bce_with_logits(logits, labels)
    if cot is not None:
        for l in range(spec.L):
            loss += float((outs[l]["X"] * cot[l]["X"]).sum())
            for e in range(len(spec.events)):
                loss += float((outs[l]["S"][e] * cot[l]["S"][e]).sum())
                loss += float((outs[l]["H"][e] * cot[l]["H"][e]).sum())
    dlogits = bce_bwd(1.0)
    for b in range(B):
        bwds, h_bwd = per_sample[b]
        dflat, dws, dbs = h_bwd(np.array([[dlogits[b]]]))
        for i in range(2):
            K._acc(grads, f"head/w{i}", dws[i])
            K._acc(grads, f"head/b{i}", dbs[i])
        dx = dflat.reshape(spec.n_ctx, spec.d)
        ds = [np.zeros((lengths[e][b], spec.ev_d(e))) for e in range(len(spec.events))]
        dh = [None] * len(spec.events)
        for l in reversed(range(spec.L)):
            if cot is not None:
                dx = dx + cot[l]["X"][b]
                ds = [ds[e] + cot[l]["S"][e][b, : lengths[e][b]] for e in range(len(spec.events))]
                dh = [(cot[l]["H"][e][b] if dh[e] is None else dh[e] + cot[l]["H"][e][b])
                      for e in range(len(spec.events))]
            dx, ds, dh_prev, gr = bwds[l](dx, ds, dh)
            K.merge_grads(grads, gr)
            dh = dh_prev
        dX_all[b] = dx
        for e in range(len(spec.events)):
            dS_all[e][b, : lengths[e][b]] = ds[e]
            if cot is not None:
                # padding rows are identity through every layer
                for l in range(spec.L):
                    dS_all[e][b, lengths[e][b]:] += cot[l]["S"][e][b, lengths[e][b]:]
    for name in p:
        if name not in grads:
            grads[name] = np.zeros_like(p[name])
    return {"loss": loss, "logits": logits, "outs": outs, "grads": grads, "dX": dX_all, "dS": dS_all}
