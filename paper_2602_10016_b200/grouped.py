"""Event-level personalization executed grouped over event types.

The reference runs one stack of modules per event type (SPEC.md:456-459,
517-518; model forward loops over events).  When the event types share one
shape (T, w, budget, seeds, rank, width, heads, depth) their sequences are
stacked along the batch — sample ``e * B + b`` is event ``e``'s sample ``b``
— and every per-event operator becomes ONE launch over all event types:

* weight generation: one GEMM batched over events, the (B, n_sum*d)
  non-sequence summary broadcast against each event's stacked ``kgv``;
* the per-sample fold (Kt = K W_q, Vt = V W_out^T) writes each event's
  slice of the grouped (E*B, H*n_kv, d) operands (one GEMM per event: its
  weights differ per event *and* per head, two batch dims already);
* the fused GDPA, sliding-window attention and HSP pooling kernels take the
  stacked batch as is (per-sample kernels; HSP reads each sample's query set
  by ``q_group``, kl_hsp_args);
* every projection (QKV, output, value, SumKronLinear) is a GEMM batched
  over the event dim against the events' weight blocks viewed as one stacked
  tensor (Params.stacked: each layer creates its events' parameters in the
  same order, so the blocks are uniformly spaced).

Parameters keep the per-event registry names and layout, so the grouped and
per-event paths are interchangeable (tests/test_gpu_grouped.py checks them
against each other and against the oracle)."""

from __future__ import annotations

import torch

from . import functional as F
from ._capi import gemm
from .tensor import flag_nonfinite, numerics_check_mode


def uniform_events(cfg) -> bool:
    """Event types that can run as one group: identical shapes everywhere the
    per-event operators differ, and the default (non-ablation) operators."""
    evs = cfg.events
    if len(evs) < 2 or cfg.pffn != "gdpa" or cfg.summarizer != "hsp" or cfg.attention != "window":
        return False
    key = lambda e: (evs[e].T, evs[e].w, evs[e].causal, evs[e].budget, evs[e].n_seeds, evs[e].rank,
                     cfg.ev_d(e), cfg.ev_heads(e), cfg.ev_layers(e), cfg.ev_acts(e))
    k0 = key(0)
    return all(key(e) == k0 for e in range(1, len(evs))) and cfg.ev_d(0) == cfg.d and cfg.ev_layers(0) == cfg.L


class FoldSpec:
    """The weight-generation blocks (kgv, wq, wout) of E event types of one
    shape (E = 1: a single event's GDPA)."""

    def __init__(self, P, wg):
        self.P = P
        self.E = len(wg)
        g0 = wg[0]
        self.H, self.n_kv, self.d_h, self.d = g0.heads, g0.n_kv, g0.head_dim, g0.dim
        self.kgv = tuple(g.kgv for g in wg)
        self.wq = tuple(g.wq for g in wg)
        self.gwout = tuple(g.wout for g in wg)


class EventGroup(FoldSpec):
    """Stacked parameter keys of one layer's grouped event types."""

    def __init__(self, P, lp):
        wg, mh, sm = lp.wg, lp.mha, lp.summ
        super().__init__(P, wg)
        m0, s0 = mh[0], sm[0]
        self.wqkv = tuple(m.wqkv for m in mh)
        self.mwout = tuple(m.wout for m in mh)
        hs = [s.hsp for s in sm]
        self.split = s0.split
        self.n_seeds, self.rank = hs[0].n_seeds, hs[0].rank
        self.h_wqkv = tuple(h.attn.wqkv for h in hs)
        self.h_wout = tuple(h.attn.wout for h in hs)
        self.zs = tuple(h.zs for h in hs)
        self.ws = tuple(h.ws for h in hs)
        self.c_wqkv = tuple(s.cls_attn.wqkv for s in sm) if s0.cls_queries else ()
        self.c_wout = tuple(s.cls_attn.wout for s in sm) if s0.cls_queries else ()

    def ok(self) -> bool:
        keys = [self.kgv, self.wq, self.gwout, self.wqkv, self.mwout, self.h_wqkv, self.h_wout, self.zs, self.ws]
        keys += [k for k in (self.c_wqkv, self.c_wout) if k]
        return all(self.P.stacked(k) is not None for k in keys)

    def value_ref(self, keys) -> F.SRef:
        """(E, H, d_h, d) value projections of stacked (3 H d_h, d) blocks."""
        H, d_h, d, E = self.H, self.d_h, self.d, self.E
        lo = 2 * H * d_h
        return F.SRef(self.P, keys, lambda w: w[:, lo:lo + H * d_h].view(E, H, d_h, d))


# ---------------------------------------------------------------------------
class _GroupFold(torch.autograd.Function):
    """Kt[e, b, h] = K[e, b, h] W_q[e, h], Vt[e, b, h] = V[e, b, h] W_out[e][:, h]^T
    (gdpa.py:120-138 per event) into the grouped (E*B, H*n_kv, d) operands of
    the fused GDPA kernels; VJP per event: dK = dKt W_q^T, dW_q += sum_b K^T dKt
    (likewise V / W_out)."""

    @staticmethod
    def forward(ctx, kv, flat, grp):
        E, B = kv.shape[0], kv.shape[1]
        H, n_kv, d_h, d = grp.H, grp.n_kv, grp.d_h, grp.d
        P = grp.P
        kv6 = kv.view(E, B, 2, H, n_kv, d_h)
        kt = torch.empty(E * B, H * n_kv, d, device=kv.device, dtype=kv.dtype)
        vt = torch.empty_like(kt)
        kt5, vt5 = kt.view(E, B, H, n_kv, d), vt.view(E, B, H, n_kv, d)
        for e in range(E):
            gemm(kv6[e, :, 0], P.w(grp.wq[e]).view(H, d_h, d), kt5[e])
            gemm(kv6[e, :, 1], P.w(grp.gwout[e]).view(d, H, d_h).permute(1, 2, 0), vt5[e])
        ctx.grp = grp
        ctx.save_for_backward(kv)
        return kt, vt

    @staticmethod
    def backward(ctx, dkt, dvt):
        (kv,) = ctx.saved_tensors
        grp = ctx.grp
        P = grp.P
        E, B = kv.shape[0], kv.shape[1]
        H, n_kv, d_h, d = grp.H, grp.n_kv, grp.d_h, grp.d
        kv6 = kv.view(E, B, 2, H, n_kv, d_h)
        dkt5 = dkt.contiguous().view(E, B, H, n_kv, d)
        dvt5 = dvt.contiguous().view(E, B, H, n_kv, d)
        dkv = torch.empty_like(kv)
        dkv6 = dkv.view(E, B, 2, H, n_kv, d_h)
        for e in range(E):
            wq = P.w(grp.wq[e]).view(H, d_h, d)
            wo = P.w(grp.gwout[e]).view(d, H, d_h).permute(1, 2, 0)
            gemm(dkt5[e], wq.transpose(1, 2), dkv6[e, :, 0])
            gemm(dvt5[e], wo.transpose(1, 2), dkv6[e, :, 1])
            with F._DwFork((kv, dkt5, dvt5)):
                gemm(kv6[e, :, 0].transpose(2, 3), dkt5[e], P.g(grp.wq[e]).view(1, H, d_h, d), beta=1.0,
                     reduce=(True, False))
                gemm(kv6[e, :, 1].transpose(2, 3), dvt5[e],
                     P.g(grp.gwout[e]).view(d, H, d_h).permute(1, 2, 0).unsqueeze(0), beta=1.0,
                     reduce=(True, False))
        return dkv, None, None


def generate_fold(xsum, grp: FoldSpec):
    """All event types' generated weights (one GEMM: the flattened summary
    broadcast against the stacked kgv blocks), folded per event into the
    (E*B, H*n_kv, d) Kt / Vt of the fused GDPA kernels (generate_kv + fold_kv,
    gdpa.py:103-138, without the per-head K / V slices' gradient copies)."""
    B = xsum.shape[0]
    flat = xsum.reshape(B, -1)
    kv = F.mm(flat, F.SRef(grp.P, grp.kgv, lambda w: w.transpose(1, 2)))  # (E, B, 2 H n_kv d_h)
    return _GroupFold.apply(kv, grp.P.flat, grp)


def window_attention(s, grp: EventGroup, lens, w: int, causal: bool):
    """mha_window (attention.py:124-129) of every event type: grouped QKV and
    output projections around one banded-attention launch over E*B samples."""
    EB, T, d = s.shape
    E = grp.E
    stash = F.ResidualStash()
    sv = s.view(E, EB // E * T, d)
    qkv = F.linear(sv, grp.P, grp.wqkv, stash_in=stash)
    o = F.swa_core(qkv.view(EB, T, 3 * d), lens, grp.H, grp.d_h, w, causal)
    y = F.linear(o.view(E, EB // E * T, d), grp.P, grp.mwout, residual=sv, stash_out=stash)
    return y.view(EB, T, d)


def summarize(S, grp: EventGroup, lens, q_rows, sink=None):
    """hsp_summarize (seqsum.py:199-210) of every event type: one pooling
    launch (each sample pools with its event's query set) and grouped value /
    output / SumKronLinear GEMMs; returns the stacked (E*B, budget, d) rows."""
    EB, T, d = S.shape
    E, H = grp.E, grp.H
    Bg = EB // E
    n_s, n_cls, n_rec = grp.n_seeds, grp.split.n_cls, grp.split.n_recent
    n_tok, k = grp.split.n_tokens, grp.rank
    splits = (n_s * H, n_cls * H) if n_cls > 0 else (n_s * H,)
    outs = F.hsp_pool(S, q_rows, lens, splits, n_recent=n_rec, sink=sink)
    P = grp.P
    v = F.head_proj(outs[0].view(EB, n_s, H, d), grp.value_ref(grp.h_wqkv))  # (EB, n_s, d)
    hseed = F.linear(v.view(E, Bg * n_s, d), P, grp.h_wout)  # (E, Bg n_s, d)
    u = F.mm(F.SRef(P, grp.zs, lambda z: z.view(E, 1, n_tok * k, n_s)), hseed.view(E, Bg, n_s, d))
    hsp_tok = F.mm(u.view(E, Bg * n_tok, k * d), F.SRef(P, grp.ws, lambda w: w.view(E, k * d, d)))
    parts = []
    if n_cls > 0:
        vc = F.head_proj(outs[1].view(EB, n_cls, H, d), grp.value_ref(grp.c_wqkv))
        parts.append(F.linear(vc.view(E, Bg * n_cls, d), P, grp.c_wout).view(EB, n_cls, d))
    parts.append(hsp_tok.view(EB, n_tok, d))
    if n_rec > 0:
        parts.append(outs[len(splits)])
    rows = F.cat_rows(parts)
    if numerics_check_mode() == "eager":
        flag_nonfinite(rows, "hsp_summarize (grouped)")
    return rows


def stage(tensors):
    """Copies of equally shaped tensors as adjacent slices of one buffer
    (so ``stack_inputs`` views them without a copy per step)."""
    buf = torch.stack([t.detach() for t in tensors])
    return list(buf.unbind(0))


def stack_inputs(S_list):
    """The events' sequences as one (E*B, T, d) batch: a view when they are
    already adjacent slices of one buffer (TrainStep stages them so), else a
    copy (autograd-tracked)."""
    s0 = S_list[0]
    n = s0.numel()
    adjacent = (all(s.shape == s0.shape and s.dtype == s0.dtype and s.is_contiguous() for s in S_list)
                and all(s.untyped_storage().data_ptr() == s0.untyped_storage().data_ptr() for s in S_list)
                and all(s.storage_offset() == s0.storage_offset() + e * n for e, s in enumerate(S_list))
                and not any(s.requires_grad for s in S_list))
    E = len(S_list)
    if adjacent:
        return s0.as_strided((E * s0.shape[0],) + tuple(s0.shape[1:]), (s0.stride(0),) + tuple(s0.stride()[1:]))
    return torch.cat(list(S_list), dim=0)
