"""FLOPs ledger and MFU, single source
of truth for the bench.

Convention (PaLM, cited by PAPER.md:77): count matmul MACs
only, 1 MAC = 2 FLOPs, training = 3 x forward.  Two ledgers:

* ``reference`` — the matmuls of the reference formulation
  (gdpa.py:120-138, attention.py:69-93/142-145, seqsum.py:26-122,
  interaction.py:106-157), band support (not dense T^2) for the window.
* ``executed`` — the matmuls the B200 path actually launches (folded GDPA,
  reassociated HSP pooling, SumKronLinear as two GEMMs), honouring CompSkip
  and liveness pruning.  This is the MFU numerator; FLOPs removed by
  reassociation are never claimed.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from .attention import band_support_sizes
from .interaction import ExpertPartition
from .seqsum import SummarySplit


def _support(T: int, w: int, causal: bool, length: int | None = None) -> int:
    L = T if length is None else length
    return int(band_support_sizes(L, w, causal).sum()) if L > 0 else 0


def layer_macs(cfg, flags, live_seq: bool = True, formulation: str = "executed", lengths=None, layer=None) -> dict:
    """Per-sample forward MACs of one layer, by component (per-event widths,
    heads and depths: an event whose stack ended before ``layer`` costs
    nothing; summary adapters count under "hsp")."""
    D = cfg.d
    out = {"wgen": 0, "gdpa": 0, "swa_proj": 0, "swa_core": 0, "hsp": 0, "sumkron": 0, "gi": 0}
    for e, ev in enumerate(cfg.events):
        if layer is not None and hasattr(cfg, "ev_layers") and layer >= cfg.ev_layers(e):
            continue
        d = cfg.ev_d(e) if hasattr(cfg, "ev_d") else D
        H = cfg.ev_heads(e) if hasattr(cfg, "ev_heads") else cfg.heads
        d_h = d // H
        T = ev.T if lengths is None else int(lengths[e])
        split = SummarySplit.for_budget(ev.budget)
        n_s, n_cls, n_tok = ev.n_seeds, split.n_cls, split.n_tokens
        pffn = getattr(cfg, "pffn", "gdpa")
        if live_seq and not flags.skip_pffn and pffn == "original":
            # pffn_original (gdpa.py:247-257): f = W2 act(W1 flat + b1) + b2, Y = S f^T
            hid = getattr(cfg, "pffn_hidden", 2 * d)
            out["wgen"] += cfg.n_sum * cfg.n_ctx * D + hid * cfg.n_sum * D + d * d * hid
            out["gdpa"] += T * d * d
        elif live_seq and not flags.skip_pffn:
            out["wgen"] += cfg.n_sum * cfg.n_ctx * D + 2 * cfg.n_kv * d_h * H * cfg.n_sum * D
            if formulation == "executed":
                out["gdpa"] += 2 * cfg.n_kv * d * d + 2 * T * d * H * cfg.n_kv
            else:
                out["gdpa"] += 2 * T * d * d + 2 * T * cfg.n_kv * d
        if live_seq and not flags.skip_self_attention:
            w = max(ev.T - 1, 0) if getattr(cfg, "attention", "window") == "full" else ev.w
            out["swa_proj"] += 4 * T * d * d
            out["swa_core"] += 2 * _support(ev.T, w, ev.causal and w == ev.w, T) * d
        if not flags.skip_hsp and getattr(cfg, "summarizer", "hsp") == "pma":
            n_q = n_tok + n_cls  # learnable-query PMA pooling (folded, like the CLS set), no SumKron
            if formulation == "executed":
                out["hsp"] += 2 * T * d * H * n_q + 2 * n_q * d * d
            else:
                out["hsp"] += n_q * (2 * d * d + 2 * T * d) + 2 * T * d * d
        elif not flags.skip_hsp:
            n_q = n_s + n_cls
            if formulation == "executed":
                # scores S Qt^T and pooling P^T S over all H*n_q queries, then
                # value + output projections; batch-shared query folding is
                # amortised over the batch and omitted (< 0.1%).
                out["hsp"] += 2 * T * d * H * n_q + n_q * d * d + n_q * d * d
                # U = Zp X (n_tok*k x n_s x d), then U' W_stack (k*d -> d)
                out["sumkron"] += ev.rank * (n_tok * n_s * d + n_tok * d * d)
            else:
                out["hsp"] += (n_s * d * d + 2 * T * d * d + 2 * n_s * T * d + n_s * d * d)
                if n_cls:
                    out["hsp"] += (n_cls * d * d + 2 * T * d * d + 2 * n_cls * T * d + n_cls * d * d)
                out["sumkron"] += ev.rank * (n_tok * n_s * d + n_tok * d * d)
        if not flags.skip_hsp and d != D:
            out["hsp"] += ev.budget * d * D  # summary adapter d_e -> d
    d = D
    part = ExpertPartition.contiguous(cfg.n_tot, cfg.experts)
    for a, b in part.ranges:
        n_i = b - a
        n_pairs = n_i * (n_i + 1) // 2
        gram = n_pairs * d if formulation == "executed" else n_i * n_i * d
        out["gi"] += gram + n_pairs * n_i * d + 2 * n_i * d * cfg.expert_hidden
    out["gi"] += cfg.n_ctx * cfg.n_tot * d
    return out


def model_macs(cfg, flags, live, formulation: str = "executed", lengths=None) -> dict:
    """Per-sample forward MACs of the whole model (layers + head)."""
    tot = {}
    for l in range(cfg.L):
        for k, v in layer_macs(cfg, flags[l], live[l], formulation, lengths, layer=l).items():
            tot[k] = tot.get(k, 0) + v
    tot["head"] = cfg.n_ctx * cfg.d * cfg.head_hidden + cfg.head_hidden
    tot["total"] = sum(tot.values())
    return tot


def train_flops_per_sample(cfg, flags, live, formulation: str = "executed") -> float:
    """2 FLOPs per MAC, x3 for forward + backward."""
    return 6.0 * model_macs(cfg, flags, live, formulation)["total"]


def mfu(flops_per_sample: float, samples_per_s: float, peak_tflops: float) -> float:
    """MFU = achieved FLOP/s / peak: 1e9 FLOPs x 100/s on a
    1e12 peak -> 0.1."""
    return flops_per_sample * samples_per_s / (peak_tflops * 1e12)


@dataclass(frozen=True)
class NeReport:
    """ne = cross_entropy / background_entropy (nats/sample)."""
    cross_entropy: float
    background_entropy: float
    ne: float
    ctr: float
    n: int


def normalized_entropy(labels, preds, from_logits: bool = False) -> NeReport:
    """Normalized entropy on the GPU (``kl_ne``; PAPER.md:438-446 Eq. A1-A2,
    SPEC.md:553-561 ``normalized_entropy``).  ``labels`` / ``preds`` are CUDA
    tensors of N values; ``preds`` are probabilities (clipped to
    [1e-12, 1 - 1e-12]) or, with ``from_logits``, the model's logits.  fp64
    accumulation in one block; the 4-double report is read back (one sync).
    Raises ``ValueError("degenerate background entropy")`` for all-zero /
    all-one labels, as the SPEC's error contract."""
    import torch

    from . import _capi

    y = labels.detach().reshape(-1).float().contiguous()
    p = preds.detach().reshape(-1).float().contiguous()
    if not (y.is_cuda and p.is_cuda):
        raise ValueError("normalized_entropy: labels and preds must be CUDA tensors (no CPU path)")
    if y.numel() < 1 or y.numel() != p.numel():
        raise ValueError("normalized_entropy: need N >= 1 labels and predictions")
    out = torch.empty(4, device=y.device, dtype=torch.float64)
    _capi.call("kl_ne", y.numel(), 1 if from_logits else 0, C.c_void_p(p.data_ptr()), C.c_void_p(y.data_ptr()),
               C.c_void_p(out.data_ptr()), _capi._stream())
    ce, h, ne, ctr = out.tolist()
    if not h > 0.0:
        raise ValueError("degenerate background entropy")
    return NeReport(ce, h, ne, ctr, int(y.numel()))
