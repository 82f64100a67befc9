"""Multi-head attention on B200: sliding-window / full self-attention and the
batch-shared-query cross-attention used by the summarizers.

Mirrors /root/reference/pkg/src/kunlun/attention.py (names, dataclasses,
validation, registry names).  Self-attention runs as: one fused QKV
projection GEMM, the banded flash kernel (tiles outside ``|i-j| <= w`` are
never visited), and the output-projection GEMM with the residual fused into
its epilogue.  Padding rows (``i >= length``) are masked as keys and come out
residual-only, exactly as attention.py:115-129.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from . import functional as F
from .tensor import Params, ShapeError, flag_nonfinite, numerics_check_mode


@dataclass
class MhaParams:
    """Per-head Q/K/V projections (d -> d_h) and output map (d -> d)
    (attention.py:24-54), packed on device as ``wqkv`` (3*H*d_h, d) =
    [w_q^0..w_q^{H-1}; w_k^0..; w_v^0..] and ``wout`` (d, d)."""

    P: Params
    prefix: str
    heads: int
    head_dim: int
    dim: int

    @property
    def wqkv(self):
        return f"{self.prefix}#wqkv"

    @property
    def wout(self):
        return f"{self.prefix}/w_out"

    @classmethod
    def create(cls, params: Params, prefix: str, dim: int, heads: int, rng: np.random.Generator | None = None,
               out_scale: float = 0.5) -> "MhaParams":
        """Same distributions and draw order as attention.py:33-46."""
        if dim % heads != 0:
            raise ValueError(f"dim {dim} not divisible by {heads} heads")
        rng = rng if rng is not None else np.random.default_rng(0)
        d_h = dim // heads
        sigma = 1.0 / np.sqrt(dim)
        p = cls(params, prefix, heads, d_h, dim)
        params.block(p.wqkv, (3 * heads * d_h, dim))
        for h in range(heads):
            for j, nm in enumerate(("w_q", "w_k", "w_v")):
                r0 = (j * heads + h) * d_h
                params.add(f"{prefix}/head{h}/{nm}", rng.normal(0.0, sigma, (d_h, dim)), block=p.wqkv,
                           index=slice(r0, r0 + d_h))
        params.add(p.wout, rng.normal(0.0, out_scale * sigma, (dim, dim)))
        return p

    def ref(self, j: int, per_head: bool = True, fp32: bool = False) -> F.PRef:
        """PRef to the Q (j=0), K (1) or V (2) projections, (H, d_h, d)."""
        H, d_h, d = self.heads, self.head_dim, self.dim
        lo = j * H * d_h
        if per_head:
            return F.PRef(self.P, self.wqkv, lambda w: w[lo: lo + H * d_h].view(H, d_h, d), fp32=fp32)
        return F.PRef(self.P, self.wqkv, lambda w: w[lo: lo + H * d_h], fp32=fp32)


@dataclass
class WindowSpec:
    """Half-window radius; position t sees keys in [t-w, t+w] (attention.py:57-66)."""

    w: int
    causal: bool = False

    def __post_init__(self):
        if self.w < 0:
            raise ValueError("window radius must be >= 0")


def band_mask(t_len: int, w: int, causal: bool = False) -> np.ndarray:
    """Boolean (T, T) support of the sliding window (attention.py:96-103)."""
    i = np.arange(t_len)[:, None]
    j = np.arange(t_len)[None, :]
    m = (j - i <= w) & (i - j <= w)
    if causal:
        m &= j <= i
    return m


def band_support_sizes(t_len: int, w: int, causal: bool = False) -> np.ndarray:
    """Keys each query attends to under the window (attention.py:132-139)."""
    i = np.arange(t_len)
    lo = np.maximum(i - w, 0)
    hi = i.copy() if causal else np.minimum(i + w, t_len - 1)
    return hi - lo + 1


def attention_macs(t_len: int, dim: int, support_total: int) -> int:
    """4 T d^2 + 2 support d (attention.py:142-145)."""
    return 4 * t_len * dim * dim + 2 * support_total * dim


def _lengths(s, lengths):
    B, T = s.shape[0], s.shape[1]
    if lengths is None:
        return torch.full((B,), T, dtype=torch.int32, device=s.device)
    if isinstance(lengths, int):
        if not 0 <= lengths <= T:
            raise ValueError(f"valid length {lengths} outside [0, {T}]")
        return torch.full((B,), lengths, dtype=torch.int32, device=s.device)
    t = torch.as_tensor(lengths).to(device=s.device, dtype=torch.int32)
    return t


def _self_attention(s, p: MhaParams, w: int, causal: bool, lengths):
    squeeze = s.dim() == 2
    if squeeze:
        s = s.unsqueeze(0)
    if s.shape[-1] != p.dim:
        raise ShapeError(f"attention needs (n, {p.dim}) inputs, got {tuple(s.shape)}")
    lens = _lengths(s, lengths)
    # the out-projection's residual gradient (dY) is added in the QKV dX epilogue
    stash = F.ResidualStash()
    qkv = F.linear(s, p.P, p.wqkv, stash_in=stash)
    o = F.swa_core(qkv, lens, p.heads, p.head_dim, w, causal)
    y = F.linear(o, p.P, p.wout, residual=s, stash_out=stash)
    if numerics_check_mode() == "eager":
        flag_nonfinite(y, "self-attention")
    return y.squeeze(0) if squeeze else y


def mha_window(s, p: MhaParams, win: WindowSpec, length=None):
    """Sliding-window self-attention plus residual (attention.py:124-129).
    ``length`` is an int or a per-sample (B,) tensor/array."""
    return _self_attention(s, p, win.w, win.causal, length)


def mha_full(s, p: MhaParams, length=None):
    """Full self-attention plus residual (attention.py:115-121) = the banded
    kernel with w >= T-1."""
    return _self_attention(s, p, max(s.shape[-2] - 1, 0), False, length)


def shared_queries(q, p: MhaParams, scale: float | None = None) -> torch.Tensor:
    """Qt_h = (q W_q^h^T) W_k^h * scale -> (H, n_q, d), fp32: the batch-shared
    reassociated query set of attention.py:85-89 (keys = S W_k^T).  It is a
    per-step (n_q x d) computation, so it stays in fp32 in every mode; only
    the T-length pooling GEMMs run in the compute dtype.  ``q`` is an fp32
    tensor or a PRef (read in fp32)."""
    H, d_h = p.heads, p.head_dim
    scale = 1.0 / np.sqrt(d_h) if scale is None else scale
    if isinstance(q, F.PRef):
        q = F.PRef(q.P, q.key, q.fn, fp32=True)
    qh = F.mm(q, F.PRef(p.P, p.wqkv, lambda w: w[: H * d_h].t(), fp32=True), p.P)  # (n_q, H*d_h)
    n_q = qh.shape[0]
    return F.mm(qh.view(n_q, H, d_h).permute(1, 0, 2), p.ref(1, fp32=True), alpha=scale)


def multi_head_attention(queries, keys_values, p: MhaParams, mask=None, lengths=None):
    """Softmax attention of query rows over key/value rows, no residual
    (attention.py:69-93).  Supported on the device path:
      * batch-shared queries ``(n_q, d)`` (or a PRef) over ``keys_values``
        ``(B, T, d)`` with per-sample ``lengths`` (mask=None) — PMA / HSP;
      * self-attention (``queries is keys_values``) with a band mask given as
        a ``WindowSpec``.
      * any other query / key rows with an explicit boolean ``mask``
        (n_q, n_k) or (B, n_q, n_k) — the reference's general form: fp32
        per-head score GEMMs, the masked row softmax kernel
        (kl_masked_softmax_*, fully-masked rows -> 0), fp32 P V, then the
        output projection in the compute dtype."""
    if isinstance(mask, WindowSpec):
        if queries is not keys_values:
            raise ValueError("windowed attention needs queries is keys_values")
        return _self_attention(keys_values, p, mask.w, mask.causal, lengths) - keys_values
    if mask is not None:
        return _masked_attention(queries, keys_values, p, mask)
    squeeze = keys_values.dim() == 2
    kv = keys_values.unsqueeze(0) if squeeze else keys_values
    qt = shared_queries(queries, p)  # (H, n_q, d)
    H, n_q = qt.shape[0], qt.shape[1]
    lens = _lengths(kv, lengths)
    q_rows = qt.transpose(0, 1).reshape(n_q * H, p.dim)  # rows (query, head)
    (pooled,) = F.hsp_pool(kv, q_rows, lens)
    o = F.head_proj(pooled.view(kv.shape[0], n_q, H, p.dim), p.ref(2))
    out = F.linear(o, p.P, p.wout)
    if numerics_check_mode() == "eager":
        flag_nonfinite(out, "multi_head_attention")
    return out.squeeze(0) if squeeze else out


def swa_support(lengths, t_len: int, w: int, causal: bool = False, heads: int = 1, d_h: int = 16):
    """Per-query key counts the SWA kernels visit (bit-exact test hook,
    kl_swa_debug_support), (B, T) int32 on the host."""
    lens = torch.as_tensor(np.asarray(lengths), dtype=torch.int32, device="cuda")
    B = lens.shape[0]
    qkv = torch.zeros(B, max(t_len, 1), 3 * heads * d_h, device="cuda", dtype=torch.float32)
    O = torch.zeros(B, max(t_len, 1), heads * d_h, device="cuda", dtype=torch.float32)
    LSE = torch.zeros(B, heads, max(t_len, 1), device="cuda", dtype=torch.float32)
    a = _capi.swa_args(qkv, lens, heads, d_h, w, causal, O, LSE)
    a.T = t_len
    sup = torch.zeros(B * max(t_len, 1), dtype=torch.int32, device="cuda")
    _capi.call("kl_swa_debug_support", C.byref(a), sup.data_ptr(), _capi._stream())
    return sup.view(B, -1)[:, :t_len].cpu().numpy()


class _MaskedSoftmax(torch.autograd.Function):
    """masked_softmax_lastdim (tensor.py:485-505) of fp32 scores (B, H, n_q,
    n_k) under a uint8 mask (n_q, n_k) or (B, H, n_q, n_k)."""

    @staticmethod
    def forward(ctx, x, mask):
        x = x.contiguous()
        y = torch.empty_like(x)
        n = x.shape[-1]
        rows = x.numel() // max(n, 1)
        _capi.call("kl_masked_softmax_fwd", rows, n, x.data_ptr(), mask.data_ptr(), mask.numel() // max(n, 1),
                   y.data_ptr(), _capi._stream())
        ctx.save_for_backward(y)
        return y

    @staticmethod
    def backward(ctx, g):
        (y,) = ctx.saved_tensors
        g = g.contiguous().float()
        dx = torch.empty_like(y)
        n = y.shape[-1]
        _capi.call("kl_masked_softmax_bwd", y.numel() // max(n, 1), n, y.data_ptr(), g.data_ptr(), dx.data_ptr(),
                   _capi._stream())
        return dx, None


def _masked_attention(queries, keys_values, p: MhaParams, mask):
    """multi_head_attention (attention.py:69-93) with an arbitrary boolean mask."""
    squeeze = keys_values.dim() == 2
    xkv = keys_values.unsqueeze(0) if squeeze else keys_values
    xq = queries.unsqueeze(0) if queries.dim() == 2 else queries
    if xq.shape[0] == 1 and xkv.shape[0] > 1:
        xq = xq.expand(xkv.shape[0], -1, -1)
    B, n_q, n_k = xkv.shape[0], xq.shape[1], xkv.shape[1]
    H, d_h, d = p.heads, p.head_dim, p.dim
    m = torch.as_tensor(np.asarray(mask) if not isinstance(mask, torch.Tensor) else mask, device=xkv.device)
    m = m.to(torch.uint8)
    if m.shape == (n_q, n_k):
        m = m.contiguous()
    elif m.shape == (B, n_q, n_k):
        m = m[:, None].expand(B, H, n_q, n_k).contiguous()
    else:
        raise ShapeError(f"mask must be ({n_q}, {n_k}) or ({B}, {n_q}, {n_k}), got {tuple(m.shape)}")
    proj = lambda x, j: F.mm(x, F.PRef(p.P, p.wqkv, lambda w, j=j: w[j * H * d_h:(j + 1) * H * d_h].t()))
    q = F.cast(proj(xq, 0), torch.float32).view(B, n_q, H, d_h).permute(0, 2, 1, 3)
    k = F.cast(proj(xkv, 1), torch.float32).view(B, n_k, H, d_h).permute(0, 2, 1, 3)
    v = F.cast(proj(xkv, 2), torch.float32).view(B, n_k, H, d_h).permute(0, 2, 1, 3)
    scores = F.mm(q, k.transpose(2, 3), alpha=1.0 / float(np.sqrt(d_h)))  # (B, H, n_q, n_k), fp32
    attn = _MaskedSoftmax.apply(scores, m)
    o = F.mm(attn, v)  # (B, H, n_q, d_h)
    cat = F.cast(o.permute(0, 2, 1, 3).reshape(B, n_q, H * d_h), xkv.dtype)
    out = F.linear(cat, p.P, p.wout)
    if numerics_check_mode() == "eager":
        flag_nonfinite(out, "multi_head_attention")
    return out.squeeze(0) if squeeze else out
