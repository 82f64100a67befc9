"""Sequence summarization on B200: PMA, Hierarchical Seed Pooling with
SumKronLinear, recent rows, and the three-part summary bundle.

Mirrors /root/reference/pkg/src/kunlun/seqsum.py (names, dataclasses,
validation, init distributions and draw order, registry names).

Execution: the seed queries (RMSNorm'd seeds, seqsum.py:96-102) and the CLS
queries (pma, seqsum.py:26-34) are batch-shared, so their key projection is
folded into the queries once per step (``Qt_h = q W_q^h^T W_k^h / sqrt(d_h)``)
and both query sets pool over S in ONE pass
(``P = softmax_t(S Qt^T)``, ``pooled = P^T S``), followed by the value and
output projections.  SumKronLinear runs as two
batched GEMMs.  Empty sequences give zeros with no gradient.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import functional as F
from .attention import MhaParams, multi_head_attention, shared_queries, _lengths
from .tensor import Params, ShapeError, flag_nonfinite, numerics_check_mode


def pma(s, queries, p: MhaParams, lengths=None):
    """Pooling by multi-head attention with learnable queries (seqsum.py:26-34)."""
    return multi_head_attention(queries, s, p, lengths=lengths)


def seed_token_bounds(n_seeds: int, n_tokens: int) -> np.ndarray:
    """Seed->token block bounds of the mean-pooling init (seqsum.py:67-71):
    float linspace truncated to int, exactly as the reference computes it."""
    return np.linspace(0, n_seeds, n_tokens + 1).astype(int)


def seed_init_base(n_seeds: int, n_tokens: int) -> np.ndarray:
    """Mean-pooling start of the token-mixing maps (seqsum.py:65-71)."""
    base = np.zeros((n_seeds, n_tokens))
    b = seed_token_bounds(n_seeds, n_tokens)
    for j in range(n_tokens):
        lo, hi = int(b[j]), max(int(b[j + 1]), int(b[j]) + 1)
        base[lo:hi, j] = 1.0 / (hi - lo)
    return base


@dataclass
class HspParams:
    """Seeds, their RMSNorm gain, the seed-attention weights and the rank-k
    compression pairs (seqsum.py:37-93).  Packed: ``zs`` (n_tokens, k, n_seeds)
    and ``ws`` (k, d, d)."""

    P: Params
    prefix: str
    attn: MhaParams
    n_seeds: int
    n_tokens: int
    rank: int
    dim: int

    def __post_init__(self):
        if self.n_seeds <= self.n_tokens:
            raise ValueError(
                f"need more seeds than output tokens for an overcomplete stage, "
                f"got {self.n_seeds} seeds for {self.n_tokens} tokens")
        if self.rank < 1:
            raise ValueError("need k >= 1 aligned (seq_map, emb_map) pairs")

    @property
    def seeds(self):
        return f"{self.prefix}/seeds"

    @property
    def gain(self):
        return f"{self.prefix}/norm_gain"

    @property
    def zs(self):
        return f"{self.prefix}#seq_maps"

    @property
    def ws(self):
        return f"{self.prefix}#emb_maps"

    @classmethod
    def create(cls, params: Params, prefix: str, dim: int, n_seeds: int, n_tokens: int, rank: int, heads: int,
               rng: np.random.Generator | None = None) -> "HspParams":
        if n_seeds <= n_tokens:
            raise ValueError("n_seeds must exceed n_tokens")
        rng = rng if rng is not None else np.random.default_rng(0)
        params.add(f"{prefix}/seeds", rng.normal(0.0, 1.0 / np.sqrt(dim), (n_seeds, dim)))
        params.add(f"{prefix}/norm_gain", np.ones(dim))
        attn = MhaParams.create(params, f"{prefix}/attn", dim, heads, rng)
        base = seed_init_base(n_seeds, n_tokens)
        p = cls(params, prefix, attn, n_seeds, n_tokens, rank, dim)
        # seq maps packed (n_tokens, k, n_seeds): as a (n_tokens*k, n_seeds)
        # matrix, row (t, i) is Z_i[:, t] (the reassociated SumKron's A operand)
        params.block(p.zs, (n_tokens, rank, n_seeds))
        params.block(p.ws, (rank, dim, dim))
        for i in range(rank):
            z = base / rank + rng.normal(0.0, 0.02, (n_seeds, n_tokens))
            w = np.eye(dim) + rng.normal(0.0, 0.02, (dim, dim))
            params.add(f"{prefix}/kron{i}/seq_map", z, block=p.zs, index=lambda v, i=i: v[:, i, :].t())
            params.add(f"{prefix}/kron{i}/emb_map", w, block=p.ws, index=i)
        return p

    def compression_param_count(self) -> int:
        return self.rank * (self.n_seeds * self.n_tokens + self.dim * self.dim)


def hsp_queries(p: HspParams) -> torch.Tensor:
    """Qt for the seed set: RMSNorm(seeds)*gain (tensor.py:552-556) folded
    through W_q, W_k (H, n_seeds, d)."""
    return shared_queries(F.rms_norm_param(p.P, p.seeds, p.gain), p.attn)


def sumkronlinear(x: torch.Tensor, p: HspParams) -> torch.Tensor:
    """Y = sum_i Z_i^T X W_i (seqsum.py:105-122) on (B, n_seeds, d),
    in the reference's order sum_i (Z_i^T X) W_i: U = Zp X per sample (Zp rows
    (t, i) = Z_i[:, t]; M = n_tokens*k), then one GEMM of the rows
    (b, t) of U, (B*n_tokens, k*d), with the stacked W_i (k*d, d)."""
    if x.shape[-2] != p.n_seeds or x.shape[-1] != p.dim:
        raise ShapeError(f"map shapes incompatible with input {tuple(x.shape)}")
    squeeze = x.dim() == 2
    if squeeze:
        x = x.unsqueeze(0)
    B = x.shape[0]
    k, n_tok, n_s, d = p.rank, p.n_tokens, p.n_seeds, p.dim
    u = F.mm(F.PRef(p.P, p.zs, lambda z: z.view(n_tok * k, n_s)), x)  # (B, n_tok*k, d)
    y = F.mm(u.view(B * n_tok, k * d), F.PRef(p.P, p.ws, lambda w: w.view(k * d, d)))
    y = y.view(B, n_tok, d)
    return y.squeeze(0) if squeeze else y


def hsp_seed_attend(s, p: HspParams, lengths=None):
    """MHA(RMSNorm(E)*g, S, S), zeros for empty sequences (seqsum.py:96-102)."""
    kv = s.unsqueeze(0) if s.dim() == 2 else s
    out = multi_head_attention(F.rms_norm_param(p.P, p.seeds, p.gain), kv, p.attn, lengths=lengths)
    return out.squeeze(0) if s.dim() == 2 else out


@dataclass
class SummarySplit:
    """Token budget split (seqsum.py:125-145)."""

    n_cls: int
    n_tokens: int
    n_recent: int

    def __post_init__(self):
        if min(self.n_cls, self.n_tokens, self.n_recent) < 0 or self.n_tokens < 1:
            raise ValueError("split counts must be >= 0 with at least one compressed token")

    @property
    def total(self) -> int:
        return self.n_cls + self.n_tokens + self.n_recent

    @classmethod
    def for_budget(cls, budget: int) -> "SummarySplit":
        q = budget // 4
        return cls(q, budget - 2 * q, q)


@dataclass
class SummaryBundle:
    """[CLS | compressed seeds | recent] (seqsum.py:148-162), each (B, n, d)."""

    cls_tokens: torch.Tensor
    hsp_tokens: torch.Tensor
    recent_tokens: torch.Tensor

    def rows(self) -> torch.Tensor:
        parts = [t for t in (self.cls_tokens, self.hsp_tokens, self.recent_tokens) if t.shape[-2] > 0]
        if len(parts) == 1:
            return parts[0]
        if parts[0].dim() == 3 and parts[0].is_cuda:
            return F.cat_rows(parts)  # one kl_regroup launch each way
        return torch.cat(parts, dim=-2)

    @property
    def total_rows(self) -> int:
        return self.cls_tokens.shape[-2] + self.hsp_tokens.shape[-2] + self.recent_tokens.shape[-2]


@dataclass
class SummarizerParams:
    """Everything for one event type's SummaryBundle (seqsum.py:165-183).

    ``mode="pma"`` is the "w/o HSP (use PMA)" ablation of PAPER.md Table 2
    (lines 355-381; PMA = MHA(Q_learnable, S, S)): the
    n_tokens middle rows are pooled by learnable queries
    (``{prefix}/pma_queries`` with ``{prefix}/pma_attn``) instead of seed
    attention + SumKronLinear."""

    hsp: HspParams | None
    cls_queries: str | None
    cls_attn: MhaParams | None
    split: SummarySplit
    mode: str = "hsp"
    pma_queries: str | None = None
    pma_attn: MhaParams | None = None

    @property
    def P(self) -> Params:
        return self.hsp.P if self.hsp is not None else self.pma_attn.P

    @classmethod
    def create(cls, params: Params, prefix: str, dim: int, split: SummarySplit, n_seeds: int, rank: int,
               heads: int, rng: np.random.Generator | None = None, mode: str = "hsp") -> "SummarizerParams":
        rng = rng if rng is not None else np.random.default_rng(0)
        if mode not in ("hsp", "pma"):
            raise ValueError(f"summarizer mode must be 'hsp' or 'pma', got {mode!r}")
        hsp = None
        if mode == "hsp":
            hsp = HspParams.create(params, f"{prefix}/hsp", dim, n_seeds, split.n_tokens, rank, heads, rng)
        queries = attn = None
        if split.n_cls > 0:
            queries = params.add(f"{prefix}/cls_queries", rng.normal(0.0, 1.0 / np.sqrt(dim), (split.n_cls, dim)))
            attn = MhaParams.create(params, f"{prefix}/cls_attn", dim, heads, rng)
        pq = pa = None
        if mode == "pma":
            pq = params.add(f"{prefix}/pma_queries", rng.normal(0.0, 1.0 / np.sqrt(dim), (split.n_tokens, dim)))
            pa = MhaParams.create(params, f"{prefix}/pma_attn", dim, heads, rng)
        return cls(hsp, queries, attn, split, mode, pq, pa)


def recent_rows(s, n_recent: int, lengths=None):
    """Last n_recent valid rows, zero-padded at the front (seqsum.py:186-196)."""
    squeeze = s.dim() == 2
    ss = s.unsqueeze(0) if squeeze else s
    out = F.recent_rows(ss, _lengths(ss, lengths), n_recent)
    return out.squeeze(0) if squeeze else out


def summary_queries(p: SummarizerParams) -> torch.Tensor:
    """The folded seed + CLS query rows ((n_seeds + n_cls) * H, d) fp32 that
    pool over S in hsp_summarize, rows ordered (query, head): each pooled set
    is (B, n, H, d) and its projections run on B*n flattened rows."""
    hp = p.hsp
    H, d = hp.attn.heads, hp.dim
    qs = hsp_queries(hp)  # (H, n_s, d)
    if p.split.n_cls > 0:
        qc = shared_queries(F.PRef(hp.P, p.cls_queries), p.cls_attn)  # (H, n_cls, d)
        qs = torch.cat([qs, qc], dim=1)
    return qs.transpose(0, 1).reshape(qs.shape[1] * H, d)


def hsp_summarize(s, p: SummarizerParams, lengths=None, sink=None, q_rows=None) -> SummaryBundle:
    """Full three-part summary [CLS | compressed seeds | recent]
    (seqsum.py:199-210).  The seed and CLS query sets pool over S in a single
    kernel pass; the recent rows come from the same op, and ``sink`` (a
    functional.GradSink) lets its S gradient accumulate into the buffer of
    the sequence's other consumers."""
    squeeze = s.dim() == 2
    S = s.unsqueeze(0) if squeeze else s
    B, T, d = S.shape
    lens = _lengths(S, lengths)
    if p.mode == "pma":
        return _pma_summarize(S, p, lens, squeeze)
    hp = p.hsp
    H = hp.attn.heads
    n_s = hp.n_seeds
    n_cls = p.split.n_cls
    if q_rows is None:  # (the model folds every layer's queries at once: functional.query_folds)
        q_rows = summary_queries(p)
    splits = (n_s * H, n_cls * H) if n_cls > 0 else (n_s * H,)
    n_rec = p.split.n_recent
    outs = F.hsp_pool(S, q_rows, lens, splits, n_recent=n_rec, sink=sink)
    pooled = outs[:len(splits)]
    hseed = F.linear(F.head_proj(pooled[0].view(B, n_s, H, d), hp.attn.ref(2)), hp.P, hp.attn.wout)
    hsp_tok = sumkronlinear(hseed, hp)
    if n_cls > 0:
        cls_tok = F.linear(F.head_proj(pooled[1].view(B, n_cls, H, d), p.cls_attn.ref(2)), hp.P, p.cls_attn.wout)
    else:
        cls_tok = S.new_zeros(B, 0, d)
    rec = outs[len(splits)] if n_rec > 0 else S.new_zeros(B, 0, d)
    bundle = SummaryBundle(cls_tok, hsp_tok, rec)
    if numerics_check_mode() == "eager":
        for t in (cls_tok, hsp_tok, rec):
            flag_nonfinite(t, "hsp_summarize")
    if squeeze:
        bundle = SummaryBundle(cls_tok[0], hsp_tok[0], rec[0])
    assert bundle.total_rows == p.split.total
    return bundle


def _pma_summarize(S, p: SummarizerParams, lens, squeeze) -> SummaryBundle:
    """[CLS | PMA(Q_learnable) | recent] (the Table 2 PMA ablation): both query
    sets pool through the batch-shared-query path (fused tcgen05 pooling)."""
    B, T, d = S.shape
    P = p.P
    cls_tok = pma(S, F.PRef(P, p.cls_queries), p.cls_attn, lens) if p.split.n_cls > 0 else S.new_zeros(B, 0, d)
    tok = pma(S, F.PRef(P, p.pma_queries), p.pma_attn, lens)
    rec = recent_rows(S, p.split.n_recent, lens) if p.split.n_recent > 0 else S.new_zeros(B, 0, d)
    if numerics_check_mode() == "eager":
        for t in (cls_tok, tok, rec):
            flag_nonfinite(t, "pma summary")
    if squeeze:
        return SummaryBundle(cls_tok[0], tok[0], rec[0])
    return SummaryBundle(cls_tok, tok, rec)
