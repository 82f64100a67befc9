"""GDPA — the personalized FFN as Generalized Dot-Product Attention, on B200.

Mirrors /root/reference/pkg/src/kunlun/gdpa.py (same names, dataclasses,
validation and registry names) over batched device tensors ``S (B, T, d)``
with per-sample ``lengths (B,)`` (int32); a single ``(T, d)`` sequence is a
batch of one.

Execution: the generated per-head K_h, V_h are folded
into the query / output projections once per sample,
``Kt_h = K_h W_q^h`` and ``Vt_h = V_h W_out,h^T`` (exact reassociation), so
the T-length work is one per-sample two-layer MLP
``Y = S + Act_h(S Kt^T / tau) Vt`` run by the GDPA core kernels
(functional.gdpa_core); rows past ``lengths`` pass through unchanged.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import functional as F
from .jagged import JaggedBatch
from .tensor import ACTIVATIONS, Params, ShapeError, flag_nonfinite, numerics_check_mode

DEFAULT_ACTIVATION_CYCLE = ("silu", "relu", "identity", "tanh")  # gdpa.py:31


@dataclass
class GdpaConfig:
    """Capacity knobs for one personalized-attention block (gdpa.py:34-69)."""

    dim: int
    heads: int
    n_kv: int = 16
    tau: float = 1.0
    activations: tuple = ()

    def __post_init__(self):
        if self.heads < 1:
            raise ValueError("need at least one head")
        if self.dim % self.heads != 0:
            raise ValueError(f"dim {self.dim} not divisible by {self.heads} heads")
        if self.n_kv < 1:
            raise ValueError("n_kv must be >= 1")
        if self.tau <= 0:
            raise ValueError("temperature must be positive")
        if not self.activations:
            cycle = DEFAULT_ACTIVATION_CYCLE
            self.activations = tuple(cycle[h % len(cycle)] for h in range(self.heads))
        if len(self.activations) != self.heads:
            raise ValueError("need one activation tag per head")
        for a in self.activations:
            if a not in ACTIVATIONS:
                raise ValueError(f"unknown activation {a!r}")

    @property
    def head_dim(self) -> int:
        return self.dim // self.heads


@dataclass
class WeightGenParams:
    """Per-head query projections, K/V generators and the output projection
    (gdpa.py:72-93), packed on device:
    ``wq`` (H*d_h, d) = [w_q^0; ...], ``kgv`` (2*H*n_kv*d_h, n_sum*d) =
    [w_kgen^0; ...; w_vgen^0; ...], ``wout`` (d, d).  Registry names
    ``{prefix}/head{h}/w_q|w_kgen|w_vgen`` and ``{prefix}/w_out`` index them."""

    P: Params
    prefix: str
    heads: int
    head_dim: int
    n_kv: int
    n_sum: int
    dim: int

    @property
    def wq(self):
        return f"{self.prefix}#wq"

    @property
    def kgv(self):
        return f"{self.prefix}#kgv"

    @property
    def wout(self):
        return f"{self.prefix}/w_out"

    @classmethod
    def create(cls, params: Params, prefix: str, cfg: GdpaConfig, n_sum: int, ctx_dim: int,
               rng: np.random.Generator | None = None, out_scale: float = 0.5) -> "WeightGenParams":
        """Same distributions and draw order as gdpa.py:83-93."""
        rng = rng if rng is not None else np.random.default_rng(0)
        H, d_h, d = cfg.heads, cfg.head_dim, cfg.dim
        fan_gen = n_sum * ctx_dim
        G = cfg.n_kv * d_h
        p = cls(params, prefix, H, d_h, cfg.n_kv, n_sum, d)
        params.block(p.wq, (H * d_h, d))
        params.block(p.kgv, (2 * H * G, fan_gen))
        for h in range(H):
            params.add(f"{prefix}/head{h}/w_q", rng.normal(0.0, 1.0 / np.sqrt(d), (d_h, d)), block=p.wq,
                       index=slice(h * d_h, (h + 1) * d_h))
            params.add(f"{prefix}/head{h}/w_kgen", rng.normal(0.0, 1.0 / np.sqrt(fan_gen), (G, fan_gen)),
                       block=p.kgv, index=slice(h * G, (h + 1) * G))
            params.add(f"{prefix}/head{h}/w_vgen", rng.normal(0.0, 1.0 / np.sqrt(fan_gen), (G, fan_gen)),
                       block=p.kgv, index=slice((H + h) * G, (H + h + 1) * G))
        params.add(p.wout, rng.normal(0.0, out_scale / np.sqrt(d), (d, d)))
        return p


def summarize_nonseq(x: torch.Tensor, pool) -> torch.Tensor:
    """X_sum = P X (gdpa.py:96-100); ``pool`` is a PRef or tensor (n_sum, n+1)."""
    n_ctx = x.shape[-2]
    pshape = pool.w().shape if isinstance(pool, F.PRef) else pool.shape
    if pshape[1] != n_ctx:
        raise ShapeError(f"pool {tuple(pshape)} does not match {n_ctx} feature rows")
    return F.mm(pool, x)


def generate_kv(x_sum: torch.Tensor, p: WeightGenParams, cfg: GdpaConfig):
    """Per-head generated K, V (gdpa.py:103-112), batched: each
    (B, H, n_kv, d_h), K_h[b] = reshape(KG_h flat(X_sum[b]), (n_kv, d_h))."""
    B = x_sum.shape[0]
    flat = x_sum.reshape(B, -1)
    kv = F.linear(flat, p.P, p.kgv)  # (B, 2*H*n_kv*d_h)
    kv = kv.view(B, 2, p.heads, p.n_kv, p.head_dim)
    return kv[:, 0], kv[:, 1]


def fold_kv(k: torch.Tensor, v: torch.Tensor, p: WeightGenParams):
    """Kt_h = K_h W_q^h, Vt_h = V_h W_out[:, h]^T -> (B, H*n_kv, d) each."""
    H, d_h, d = p.heads, p.head_dim, p.dim
    B = k.shape[0]
    kt = F.mm(k, F.PRef(p.P, p.wq, lambda w: w.view(H, d_h, d)))
    vt = F.mm(v, F.PRef(p.P, p.wout, lambda w: w.view(d, H, d_h).permute(1, 2, 0)))
    return kt.reshape(B, H * p.n_kv, d), vt.reshape(B, H * p.n_kv, d)


def _lengths(s: torch.Tensor, lengths):
    B, T = s.shape[0], s.shape[1]
    if lengths is None:
        return torch.full((B,), T, dtype=torch.int32, device=s.device)
    if isinstance(lengths, torch.Tensor):
        return lengths.to(device=s.device, dtype=torch.int32)
    return torch.as_tensor(np.asarray(lengths), dtype=torch.int32, device=s.device)


def gdpa_forward(s: torch.Tensor, x_sum: torch.Tensor, cfg: GdpaConfig, p: WeightGenParams, kv=None,
                 lengths=None) -> torch.Tensor:
    """Attention-style personalized FFN plus residual (gdpa.py:120-138)."""
    squeeze = s.dim() == 2
    if squeeze:
        s = s.unsqueeze(0)
        x_sum = x_sum.unsqueeze(0)
    if s.shape[-1] != cfg.dim:
        raise ShapeError(f"sequence must be (T, {cfg.dim}), got {tuple(s.shape)}")
    if kv is None:
        kv = generate_kv(x_sum, p, cfg)
    kt, vt = fold_kv(kv[0], kv[1], p)
    y = F.gdpa_core(s, kt, vt, _lengths(s, lengths), cfg.activations, cfg.n_kv, 1.0 / cfg.tau)
    if numerics_check_mode() == "eager":
        flag_nonfinite(y, "gdpa_forward")
    return y.squeeze(0) if squeeze else y


def gdpa_forward_blockwise(s, x_sum, cfg: GdpaConfig, p: WeightGenParams, block_t=None, block_kv=None, kv=None,
                           lengths=None):
    """Streaming-tile variant (gdpa.py:190-206).  The device kernels always
    tile (T in 128-row tiles, all n_kv columns of a head in one pass); the
    reference's tile sizes only affect its Python loop, so they are accepted
    and validated but do not change the result (<= 1e-10 in the reference)."""
    if (block_t is not None and block_t < 1) or (block_kv is not None and block_kv < 1):
        raise ValueError("tile sizes must be >= 1")
    return gdpa_forward(s, x_sum, cfg, p, kv=kv, lengths=lengths)


def gdpa_forward_jagged(batch: JaggedBatch, x_sums, cfg: GdpaConfig, p: WeightGenParams, block_t=None,
                        block_kv=None) -> JaggedBatch:
    """Per-sample GDPA over a jagged batch (gdpa.py:209-224) as ONE batched
    launch on the padded layout; zero-length samples pass through."""
    if len(x_sums) != batch.batch_size:
        raise ShapeError("need one context summary per sample")
    padded, _ = batch.to_padded()
    lengths = batch.lengths()
    device, dtype = p.P.device, p.P.compute_dtype
    s = torch.as_tensor(padded, dtype=dtype, device=device)
    xs = torch.stack([torch.as_tensor(np.asarray(x), dtype=dtype, device=device) for x in x_sums])
    with torch.no_grad():
        y = gdpa_forward_blockwise(s, xs, cfg, p, block_t, block_kv, lengths=lengths)
    out = y.float().cpu().numpy().astype(np.float64)
    values = np.concatenate([out[i, : lengths[i]] for i in range(batch.batch_size)], axis=0)
    ts = None if batch.timestamps is None else batch.timestamps.copy()
    return JaggedBatch(values, batch.offsets.copy(), ts)


# ---------------------------------------------------------------------------
# "w/o GDPA" ablation baseline (Table 2): the original PFFN


@dataclass
class PffnParams:
    """Two-layer MLP emitting a (d, d) rowwise transform from the summary
    (gdpa.py:227-245): registry names ``{prefix}/w1, b1, w2, b2``, the
    reference's init distributions and draw order."""

    P: Params
    prefix: str
    dim: int
    hidden: int
    hidden_act: str = "silu"

    @property
    def w1(self):
        return f"{self.prefix}/w1"

    @property
    def b1(self):
        return f"{self.prefix}/b1"

    @property
    def w2(self):
        return f"{self.prefix}/w2"

    @property
    def b2(self):
        return f"{self.prefix}/b2"

    @classmethod
    def create(cls, params: Params, prefix: str, dim: int, n_sum: int, ctx_dim: int, hidden: int,
               rng: np.random.Generator | None = None) -> "PffnParams":
        rng = rng if rng is not None else np.random.default_rng(0)
        fan = n_sum * ctx_dim
        p = cls(params, prefix, dim, hidden)
        params.add(p.w1, rng.normal(0.0, 1.0 / np.sqrt(fan), (hidden, fan)))
        params.add(p.b1, np.zeros(hidden))
        params.add(p.w2, rng.normal(0.0, 0.1 / np.sqrt(hidden), (dim * dim, hidden)))
        params.add(p.b2, np.zeros(dim * dim))
        return p


def pffn_original(x_sum: torch.Tensor, s: torch.Tensor, p: PffnParams, lengths=None) -> torch.Tensor:
    """Original formulation (gdpa.py:247-257): per sample f = reshape(W2
    act(W1 flat(X_sum) + b1) + b2, (d, d)), Y = S f^T — no residual (the
    non-stackable baseline kept for ablation).  Batched: two bias / activation
    GEMM epilogues for f, one batched GEMM for Y."""
    squeeze = s.dim() == 2
    if squeeze:
        s, x_sum = s.unsqueeze(0), x_sum.unsqueeze(0)
    B, d = s.shape[0], s.shape[-1]
    if d != p.dim:
        raise ShapeError(f"sequence width {d} does not match the PFFN dim {p.dim}")
    flat = x_sum.reshape(B, -1)
    h = F.linear(flat, p.P, p.w1, p.b1, act=p.hidden_act)
    f = F.linear(h, p.P, p.w2, p.b2).view(B, d, d)
    y = F.mm(s, f.transpose(1, 2))
    if lengths is not None:  # padding rows pass through (the reference sees only the valid rows)
        y = F.rows_select(y, s, _lengths(s, lengths))
    if numerics_check_mode() == "eager":
        flag_nonfinite(y, "pffn_original")
    return y.squeeze(0) if squeeze else y
