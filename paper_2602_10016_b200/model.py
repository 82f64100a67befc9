"""Kunlun model assembly on B200: event configs, CompSkip (Alg. 4), the
layer forward (Alg. 1) and the prediction head.

The reference ships no ``model`` module; this follows
SPEC.md:451-533 and PAPER.md:515-541 / 586-603 exactly as SURVEY.md
Appendix A.1 pins the composition (the oracle's ``oracle/model.py`` restates
the same order).  CompSkip is host-side kernel selection: a skipped
sub-module launches nothing.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import functional as F
from . import grouped
from .attention import MhaParams, WindowSpec, mha_full, mha_window
from .gdpa import GdpaConfig, PffnParams, WeightGenParams, pffn_original, summarize_nonseq
from .interaction import ExpertPartition, InteractionParams, global_interaction
from .mlp import Mlp
from .seqsum import SummarizerParams, SummarySplit, hsp_summarize, summary_queries
from .tensor import Params, ShapeError, _flag, flag_nonfinite, numerics_check_mode

DEFAULT_ACTIVATION_CYCLE = ("silu", "relu", "identity", "tanh")
FOLD_ALL_LAYERS = True  # fold every layer's HSP/CLS queries in one batched pass (tests A/B it)


@dataclass
class EventConfig:
    """Per-event sequence knobs: padded length T, window
    half-width w, summary token budget, HSP seeds and SumKron rank, and the
    event's own width ``d``, heads and depth ``layers`` (0 = the model's;
    event-level personalization: an event with fewer layers
    holds its last summaries for the deeper global layers, and a learnable
    linear adapter maps its summaries to the model width when d != d_model)."""

    T: int
    w: int
    budget: int
    n_seeds: int
    rank: int
    causal: bool = False
    name: str = ""
    d: int = 0
    heads: int = 0
    layers: int = 0

    def __post_init__(self):
        if min(self.T, self.budget, self.n_seeds, self.rank) < 1 or self.w < 0:
            raise ValueError("event config values must be positive")
        if min(self.d, self.heads, self.layers) < 0:
            raise ValueError("event width / heads / layers must be >= 0 (0 = the model's)")


@dataclass
class LayerSkipFlags:
    """Alg. 4 per-layer flags."""

    skip_self_attention: bool = False
    skip_hsp: bool = False
    skip_pffn: bool = False

    def as_tuple(self):
        return (self.skip_self_attention, self.skip_hsp, self.skip_pffn)


def compskip_config(L: int, enabled: bool = True) -> list:
    """Alg. 4: even l -> skip self-attention
    (fresh HSP + PFFN); odd l -> reuse H_prev and skip PFFN."""
    if L < 1:
        raise ValueError("need at least one layer")
    if not enabled:
        return [LayerSkipFlags() for _ in range(L)]
    return [LayerSkipFlags(True, False, False) if l % 2 == 0 else LayerSkipFlags(False, True, True)
            for l in range(L)]


@dataclass
class ModelConfig:
    """global layers, width, heads, non-sequence tokens n+1,
    events, n_sum, n_kv, experts M, CompSkip."""

    L: int
    d: int
    heads: int
    n_ctx: int
    events: list
    n_sum: int = 4
    n_kv: int = 16
    experts: int = 2
    compskip: bool = False
    gdpa_acts: tuple = ()
    expert_hidden: int = 0
    head_hidden: int = 0
    # PAPER.md Table 2 ablations (lines 355-381): "original" = the pffn_original
    # baseline instead of GDPA (gdpa.py:227-257); "pma" = learnable-query PMA
    # summaries instead of HSP; "full" = full self-attention instead of SWA
    pffn: str = "gdpa"
    summarizer: str = "hsp"
    attention: str = "window"
    pffn_hidden: int = 0
    # event types of one shape run grouped (grouped.py): stacked along the
    # batch, one launch per operator over all of them
    group_events: bool = True

    def __post_init__(self):
        if self.d % self.heads:
            raise ValueError(f"dim {self.d} not divisible by {self.heads} heads")
        if not self.gdpa_acts:
            c = DEFAULT_ACTIVATION_CYCLE
            self.gdpa_acts = tuple(c[h % len(c)] for h in range(self.heads))
        self.expert_hidden = self.expert_hidden or 2 * self.d
        self.head_hidden = self.head_hidden or 4 * self.d
        self.pffn_hidden = self.pffn_hidden or 2 * self.d
        if self.pffn not in ("gdpa", "original") or self.summarizer not in ("hsp", "pma") or \
                self.attention not in ("window", "full"):
            raise ValueError("ablation switches: pffn gdpa|original, summarizer hsp|pma, attention window|full")
        for e in range(len(self.events)):
            if self.ev_d(e) % self.ev_heads(e):
                raise ValueError(f"event {e}: dim {self.ev_d(e)} not divisible by {self.ev_heads(e)} heads")
            if self.ev_layers(e) > self.L:
                raise ValueError(f"event {e}: {self.ev_layers(e)} layers > the model's {self.L}")
        ExpertPartition.contiguous(self.n_tot, self.experts)

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
        c = DEFAULT_ACTIVATION_CYCLE
        return tuple(c[h % len(c)] for h in range(H))

    def gdpa_cfg(self, e: int) -> GdpaConfig:
        # tau = the event's padded max length
        return GdpaConfig(self.ev_d(e), self.ev_heads(e), self.n_kv, float(self.events[e].T), self.ev_acts(e))


@dataclass
class LayerParams:
    pool: str
    wg: list
    mha: list
    summ: list
    gi: InteractionParams
    adapters: list = field(default_factory=list)  # per event: (d, d_e) block key or None


class _Boundary(torch.autograd.Function):
    """Identity on a layer's inputs whose backward fires after every
    backward kernel of that layer: the data-parallel reducer's hook point
    (dist.py) for launching that layer's gradient bucket."""

    @staticmethod
    def forward(ctx, hook, layer, *xs):
        ctx.hook, ctx.layer = hook, layer
        return xs if len(xs) > 1 else xs[0]

    @staticmethod
    def backward(ctx, *gs):
        ctx.hook(ctx.layer)
        return (None, None) + gs


class KunlunModel:
    """Parameters + batched forward of the Kunlun model on one device.

    Registry names (SURVEY.md Appendix A.3 with our layer/event prefixes):
    ``L{l}/pool``, ``L{l}/ev{e}/gdpa/...``, ``L{l}/ev{e}/mha/...``,
    ``L{l}/ev{e}/summ/...``, ``L{l}/gi/...``, ``head/w0..b1`` — identical to
    ``oracle/model.py``."""

    def __init__(self, cfg: ModelConfig, device="cuda", dtype=torch.bfloat16, seed: int = 0):
        self.cfg = cfg
        self.dtype = dtype
        rng = np.random.default_rng(seed)
        P = Params()
        self.P = P
        d, H = cfg.d, cfg.heads
        part = ExpertPartition.contiguous(cfg.n_tot, cfg.experts)
        self.layers = []
        for l in range(cfg.L):
            pool = P.add(f"L{l}/pool", rng.normal(0.0, 1.0 / np.sqrt(cfg.n_ctx), (cfg.n_sum, cfg.n_ctx)))
            wg, mh, sm, ad = [], [], [], []
            for e, ev in enumerate(cfg.events):
                if l >= cfg.ev_layers(e):  # the event's stack ended: its summaries are held (hold-last)
                    wg.append(None), mh.append(None), sm.append(None), ad.append(None)
                    continue
                de, He = cfg.ev_d(e), cfg.ev_heads(e)
                if cfg.pffn == "original":
                    wg.append(PffnParams.create(P, f"L{l}/ev{e}/pffn", de, cfg.n_sum, d, cfg.pffn_hidden, rng))
                else:
                    wg.append(WeightGenParams.create(P, f"L{l}/ev{e}/gdpa", cfg.gdpa_cfg(e), cfg.n_sum, d, rng))
                mh.append(MhaParams.create(P, f"L{l}/ev{e}/mha", de, He, rng))
                sm.append(SummarizerParams.create(P, f"L{l}/ev{e}/summ", de, SummarySplit.for_budget(ev.budget),
                                                  ev.n_seeds, ev.rank, He, rng, mode=cfg.summarizer))
                ad.append(P.add(f"L{l}/ev{e}/adapter", rng.normal(0.0, 1.0 / np.sqrt(de), (d, de)))
                          if de != d else None)
            gi = InteractionParams.create(P, f"L{l}/gi", part, cfg.n_ctx, d, cfg.expert_hidden, rng)
            self.layers.append(LayerParams(pool, wg, mh, sm, gi, ad))
        self.head = Mlp.create(P, "head", [cfg.n_ctx * d, cfg.head_hidden, 1], ["silu", "identity"], rng)
        P.finalize(device, dtype)
        self.groups = None
        if cfg.group_events and grouped.uniform_events(cfg):
            gs = [grouped.EventGroup(P, lp) for lp in self.layers]
            if all(g.ok() for g in gs):
                self.groups = gs
        if torch.device(device).type == "cuda":
            _flag(device)  # the non-finite flag exists before any CUDA-graph capture
        self.flags = compskip_config(cfg.L, cfg.compskip)
        self.layer_hook = None  # set by dist.GradReducer

    # ------------------------------------------------------------------
    def late_grad_blocks(self):
        """Block keys whose gradients are written after every layer's
        backward: the query-fold inputs (seeds, gains, query/key projections,
        CLS queries), folded once per step before layer 0 (query_rows)."""
        keys = []
        for l in range(self.cfg.L):
            if self.flags[l].skip_hsp or self.cfg.summarizer != "hsp":
                continue
            for s in self.layers[l].summ:
                if s is None:
                    continue
                keys += [s.hsp.seeds, s.hsp.gain, s.hsp.attn.wqkv]
                if s.cls_queries:
                    keys += [s.cls_queries, s.cls_attn.wqkv]
        return keys

    def layer_param_ranges(self):
        """Flat [lo, hi) parameter range of each layer (the head rides with
        the last layer)."""
        starts = [self.P.block_range(self.P.block_of(f"L{l}/pool")[0])[0] for l in range(self.cfg.L)]
        ends = starts[1:] + [self.P.gflat.numel()]
        return list(zip(starts, ends))

    def query_rows(self):
        """{(layer, event): (HQ, d) fp32 query rows} of every layer that runs
        HSP, folded for all those layers at once per event
        (functional.query_folds); {} if the layout does not allow it."""
        cfg = self.cfg
        out = {}
        layers = [l for l in range(cfg.L) if not self.flags[l].skip_hsp]
        if not layers or cfg.summarizer != "hsp":
            return out
        if self.groups is not None:  # grouped event types: per layer, every event's queries in one pass
            for l in layers:
                sp = self.layers[l].summ
                keys = ([s.hsp.seeds for s in sp], [s.hsp.gain for s in sp], [s.hsp.attn.wqkv for s in sp],
                        [s.cls_queries for s in sp] if sp[0].cls_queries else [],
                        [s.cls_attn.wqkv for s in sp] if sp[0].cls_queries else [])
                q = F.query_folds(self.P, keys, cfg.heads, cfg.d // cfg.heads, stacked=True)
                if q is None:
                    return {}
                out[l] = q  # (E, HQ, d)
            return out
        for e in range(len(cfg.events)):
            lay_e = [l for l in layers if l < cfg.ev_layers(e)]
            if not lay_e:
                continue
            sp = [self.layers[l].summ[e] for l in lay_e]
            keys = ([s.hsp.seeds for s in sp], [s.hsp.gain for s in sp], [s.hsp.attn.wqkv for s in sp],
                    [s.cls_queries for s in sp] if sp[0].cls_queries else [],
                    [s.cls_attn.wqkv for s in sp] if sp[0].cls_queries else [])
            qs = F.query_folds(self.P, keys, cfg.ev_heads(e), cfg.ev_d(e) // cfg.ev_heads(e))
            if qs is None:
                return {}
            for l, q in zip(lay_e, qs):
                out[(l, e)] = q
        return out

    def layer_forward(self, l: int, flags: LayerSkipFlags, X, S_list, lengths, H_prev, live_seq=True, qrows=None):
        """One Kunlun layer (Alg. 1), batched.  ``live_seq=False`` skips the
        sequence branch (GDPA + SWA) when its output cannot reach the loss
        (liveness pruning); the returned S' is then
        the input S."""
        cfg = self.cfg
        lp = self.layers[l]
        if flags.skip_hsp and H_prev is None:
            raise ValueError("skip_hsp on a layer without H_prev")
        if self.layer_hook is not None:
            outs = _Boundary.apply(self.layer_hook, l, X, *S_list)
            X, S_list = outs[0], list(outs[1:])
        # one shared dS buffer per event sequence: its consumers (the GDPA
        # branch, HSP pooling + recent rows) accumulate into it
        sinks = [F.GradSink() for _ in cfg.events]
        S_list = [F.seq_join(s, k) for s, k in zip(S_list, sinks)]

        events = [e for e in range(len(cfg.events)) if l < cfg.ev_layers(e)]  # events whose stack reaches l
        held = [e for e in range(len(cfg.events)) if l >= cfg.ev_layers(e)]
        if held and H_prev is None:
            raise ValueError("an event's stack ended before the first layer")

        def x_branch():  # HSP summaries (per event, parallel branches) -> global interaction
            def hsp(e):
                def run():
                    qr = qrows.get((l, e)) if qrows else None
                    rows = hsp_summarize(S_list[e], lp.summ[e], lengths[e], sink=sinks[e], q_rows=qr).rows()
                    if lp.adapters and lp.adapters[e] is not None:  # d_e -> d (learnable linear adapter)
                        rows = F.linear(rows, self.P, lp.adapters[e])
                    return rows
                return run
            if flags.skip_hsp or not events:
                H_list = list(H_prev)
            else:
                fresh = F.run_branches([hsp(e) for e in events], X.device, name="ev_x")
                H_list = list(H_prev) if H_prev is not None else [None] * len(cfg.events)
                for e, h in zip(events, fresh):
                    H_list[e] = h  # events whose stack ended keep their last summaries
            return global_interaction(X, H_list, lp.gi), H_list

        def s_branch():  # GDPA (weights generated from X) -> windowed self-attention, per event
            xsum = summarize_nonseq(X, F.PRef(self.P, lp.pool)) if (not flags.skip_pffn and live_seq) else None

            def seq(e):
                def run():
                    ev = cfg.events[e]
                    s = S_list[e]
                    if live_seq and not flags.skip_pffn and cfg.pffn == "original":
                        s = pffn_original(xsum, s, lp.wg[e], lengths[e])  # Table 2 "w/o GDPA" (no residual)
                    elif live_seq and not flags.skip_pffn:
                        kt, vt = grouped.generate_fold(xsum, grouped.FoldSpec(self.P, [lp.wg[e]]))
                        s = F.gdpa_core(s, kt, vt, lengths[e], cfg.ev_acts(e), cfg.n_kv, 1.0 / float(ev.T),
                                        sink=sinks[e])
                        if numerics_check_mode() == "eager":
                            flag_nonfinite(s, f"layer {l} event {e} GDPA")
                    if live_seq and not flags.skip_self_attention and cfg.attention == "full":
                        s = mha_full(s, lp.mha[e], lengths[e])  # Table 2 "w/o SWA"
                    elif live_seq and not flags.skip_self_attention:
                        s = mha_window(s, lp.mha[e], WindowSpec(ev.w, ev.causal), lengths[e])
                    return s
                return run
            # events are independent sequences: parallel branches; the sequence
            # of an event whose stack ended passes through unchanged
            outs = F.run_branches([seq(e) for e in events], X.device, inputs=[xsum] if xsum is not None else (),
                                  name="ev_s")
            S_new = list(S_list)
            for e, s in zip(events, outs):
                S_new[e] = s
            return S_new

        # the two branches only share their inputs: the sequence branch runs on
        # the current stream, the summary / interaction branch beside it
        # (parallel CUDA-graph branches, forward and backward).  The sequence
        # branch is issued last so its backward runs first: GDPA registers the
        # shared dS and HSP pooling accumulates into it.
        shared = [X] + list(S_list) + list(qrows.values() if qrows else []) + list(H_prev or [])
        (Xn, H_list), S_out = F.run_branches([x_branch, s_branch], X.device, inputs=shared, name="xbranch",
                                             side_first=True)
        S_out = list(S_out)
        return Xn, S_out, H_list

    def _group_queries(self, l, qrows):
        """(E, HQ, d) fp32: every event type's folded query rows of layer l."""
        E = len(self.cfg.events)
        if qrows:
            return qrows[l]
        return torch.stack([summary_queries(self.layers[l].summ[e]) for e in range(E)])

    def layer_forward_grouped(self, l: int, flags: LayerSkipFlags, X, S, lens, H_prev, live_seq=True, qrows=None):
        """layer_forward with the event types grouped (grouped.py): S is the
        (E*B, T, d) stack of every event's sequence, ``lens`` its (E*B,)
        lengths; H_prev / the returned H are per-event (B, budget, d) lists."""
        cfg = self.cfg
        lp, grp = self.layers[l], self.groups[l]
        E, B = grp.E, X.shape[0]
        ev = cfg.events[0]
        if flags.skip_hsp and H_prev is None:
            raise ValueError("skip_hsp on a layer without H_prev")
        if self.layer_hook is not None:
            X, S = _Boundary.apply(self.layer_hook, l, X, S)
        sink = F.GradSink()  # the stacked sequences' one shared gradient buffer
        S = F.seq_join(S, sink)

        def x_branch():
            if flags.skip_hsp:
                H_list = list(H_prev)
            else:
                rows = grouped.summarize(S, grp, lens, self._group_queries(l, qrows), sink=sink)
                H_list = list(rows.view(E, B, *rows.shape[1:]).unbind(0))
            return global_interaction(X, H_list, lp.gi), H_list

        def s_branch():
            s = S
            if live_seq and not flags.skip_pffn:
                kt, vt = grouped.generate_fold(summarize_nonseq(X, F.PRef(self.P, lp.pool)), grp)
                s = F.gdpa_core(s, kt, vt, lens, cfg.ev_acts(0), cfg.n_kv, 1.0 / float(ev.T), sink=sink)
                if numerics_check_mode() == "eager":
                    flag_nonfinite(s, f"layer {l} GDPA (grouped events)")
            if live_seq and not flags.skip_self_attention:
                s = grouped.window_attention(s, grp, lens, ev.w, ev.causal)
            return s

        shared = [X, S] + list(qrows.values() if qrows else []) + list(H_prev or [])
        (Xn, H_list), S_out = F.run_branches([x_branch, s_branch], X.device, inputs=shared, name="xbranch",
                                             side_first=True)
        return Xn, S_out, H_list

    def seq_live(self) -> list:
        """Layers whose sequence output can still reach a later HSP (and so
        the loss): l is live iff some l' > l does not skip HSP."""
        L = self.cfg.L
        return [any(not self.flags[j].skip_hsp for j in range(l + 1, L)) for l in range(L)]

    def forward(self, X, S_list, lengths, keep_outputs=False, prune_dead=True):
        """X (B, n+1, d), S_list[e] (B, T_e, d) in the compute dtype,
        lengths[e] (B,) int32.  Returns logits (B,) fp32 and, if asked, every
        layer's (X', S', H)."""
        live = self.seq_live() if prune_dead else [True] * self.cfg.L
        H = None
        outs = []
        qrows = None
        if FOLD_ALL_LAYERS:
            # the query folds (small fp32 products) only feed the summary
            # branches: in a training step (which joins every side stream
            # before the optimizer) issue them on that branch's stream, beside
            # layer 0's sequence branch (their backward then overlaps it too)
            if F.DW_STREAM_FWD and X.is_cuda:
                side = F.side_stream(X.device, "xbranch")
                side.wait_stream(torch.cuda.current_stream(X.device))
                with torch.cuda.stream(side):
                    qrows = self.query_rows()
            else:
                qrows = self.query_rows()
        if self.groups is not None:  # event types stacked along the batch (grouped.py)
            E = len(S_list)
            S = grouped.stack_inputs(S_list)
            lens = grouped.stack_inputs([torch.as_tensor(t, dtype=torch.int32, device=S.device) for t in lengths])
            for l in range(self.cfg.L):
                X, S, H = self.layer_forward_grouped(l, self.flags[l], X, S, lens, H, live_seq=live[l], qrows=qrows)
                if keep_outputs:
                    outs.append((X, list(S.view(E, -1, *S.shape[1:]).unbind(0)), list(H)))
        else:
            for l in range(self.cfg.L):
                X, S_list, H = self.layer_forward(l, self.flags[l], X, S_list, lengths, H, live_seq=live[l],
                                                  qrows=qrows)
                if keep_outputs:
                    outs.append((X, list(S_list), list(H)))
        B = X.shape[0]
        z = self.head.apply_rows(X.reshape(B, -1))
        logits = F.cast(z, torch.float32).reshape(B)
        flag_nonfinite(logits, "logits")  # deferred: read by raise_if_nonfinite / TrainStep.check_numerics
        return (logits, outs) if keep_outputs else logits

    def loss(self, X, S_list, lengths, labels, prune_dead=True):
        logits = self.forward(X, S_list, lengths, prune_dead=prune_dead)
        loss = F.bce_with_logits(logits, labels)
        flag_nonfinite(loss, "loss")
        return loss, logits

    def count_params(self) -> int:
        return self.P.count()
