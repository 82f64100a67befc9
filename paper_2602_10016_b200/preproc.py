"""Preprocessing — raw features to unified embeddings, the step before layer
0 (reference ``kunlun.preproc``): the schemas (``EventSchema``,
``FeatureSchema`` preproc.py:23-63), the non-sequence embedding
(``embed_dense`` / ``embed_sparse`` / ``assemble_nonseq`` preproc.py:103-127,
fused on the device into one gather kernel, ``embed_nonseq``), the
multi-sequence fusion (``fuse_sequences`` preproc.py:130-143, ``align_right``
146-152), and ROTE, the rotary temporal encoding (``RoteConfig`` preproc.py:66-100,
``temporal_angle`` 155-159, ``rote_raw`` / ``rote`` 162-172,
``gaps_from_timestamps`` 175-184, ``rote_sequence`` 187-199;
``rotate_pairs`` tensor.py:508-532).

B200 path: one ``kl_rote`` launch per direction over the padded batch
``(B, T, d)`` with per-sample ``lengths`` and ``(B, T)`` fp64 timestamps;
angles in fp64 (reduced mod 2 pi), sin/cos in fp32, forward and VJP (rotation
by the negative angles) in the same kernel.  Rows at or past a sample's length
pass through unchanged.  No CPU path: inputs must be CUDA tensors."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import _capi
from . import functional as F
from .tensor import Params, ShapeError


@dataclass
class RoteConfig:
    """Each of the d/2 planes rotates by t*pos_freqs[i] + tau*temp_freqs[i],
    tau = log(1 + delta_t / tau_scale) (preproc.py:66-100, same validation)."""

    pos_freqs: np.ndarray
    temp_freqs: np.ndarray
    tau_scale: float = 60.0
    gap_mode: str = "previous"  # or "latest"

    def __post_init__(self):
        self.pos_freqs = np.asarray(self.pos_freqs, dtype=np.float64)
        self.temp_freqs = np.asarray(self.temp_freqs, dtype=np.float64)
        if self.tau_scale <= 0:
            raise ValueError("tau_scale must be positive")
        if self.pos_freqs.shape != self.temp_freqs.shape or self.pos_freqs.ndim != 1:
            raise ValueError("frequency lists must be 1-D and equally long")
        if self.gap_mode not in ("previous", "latest"):
            raise ValueError(f"unknown gap mode {self.gap_mode!r}")
        self._dev = {}

    @classmethod
    def default(cls, dim: int, tau_scale: float = 60.0, gap_mode: str = "previous") -> "RoteConfig":
        if dim < 2 or dim % 2 != 0:
            raise ValueError("rotary encoding needs an even dim >= 2")
        half = dim // 2
        freqs = 10000.0 ** (-2.0 * np.arange(half) / dim)
        return cls(freqs, freqs.copy(), tau_scale, gap_mode)

    @property
    def half_dim(self) -> int:
        return self.pos_freqs.size

    def device_freqs(self, device) -> tuple[torch.Tensor, torch.Tensor]:
        """fp64 copies of the schedules on ``device``, uploaded once per
        (device, schedule values): reassigning pos_freqs / temp_freqs
        re-uploads.  Call it (or run one eager step) before capturing a CUDA
        graph — the upload is a host copy."""
        key = (str(device), id(self.pos_freqs), id(self.temp_freqs), self.pos_freqs.tobytes().__hash__(),
               self.temp_freqs.tobytes().__hash__())
        if key not in self._dev:
            self._dev[key] = (torch.tensor(self.pos_freqs, device=device, dtype=torch.float64),
                              torch.tensor(self.temp_freqs, device=device, dtype=torch.float64))
        return self._dev[key]


def temporal_angle(delta_t: float, cfg: RoteConfig) -> float:
    """Log-scaled gap value fed to the temporal frequencies (preproc.py:155-159)."""
    if delta_t < 0:
        raise ValueError(f"time gap must be >= 0, got {delta_t}")
    return float(np.log1p(delta_t / cfg.tau_scale))


def _launch(x, lengths, ts, cfg, inverse):
    y = torch.empty_like(x)
    a = _capi.RoteArgs()
    a.B, a.T, a.d, a.dtype = x.shape[0], x.shape[1], x.shape[2], _capi.dt(x)
    a.x, a.x_rs, a.x_bs = x.data_ptr(), x.stride(1), x.stride(0)
    a.y, a.y_rs, a.y_bs = y.data_ptr(), y.stride(1), y.stride(0)
    a.lengths = lengths.data_ptr() if lengths is not None else None
    a.timestamps = ts.data_ptr() if ts is not None else None
    a.ts_bs = ts.stride(0) if ts is not None else 0
    pf, tf = cfg.device_freqs(x.device)
    a.pos_freqs, a.temp_freqs = pf.data_ptr(), tf.data_ptr()
    a.tau_scale, a.gap_mode, a.inverse = float(cfg.tau_scale), 0 if cfg.gap_mode == "previous" else 1, int(inverse)
    _capi.call("kl_rote", C.byref(a), _capi._stream())
    return y


class _Rote(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, lengths, ts, cfg):
        ctx.cfg, ctx.lengths, ctx.ts = cfg, lengths, ts
        return _launch(x, lengths, ts, cfg, False)

    @staticmethod
    def backward(ctx, g):
        return _launch(g.contiguous(), ctx.lengths, ctx.ts, ctx.cfg, True), None, None, None


def rote_sequence(s: torch.Tensor, timestamps, cfg: RoteConfig, lengths: torch.Tensor | None = None) -> torch.Tensor:
    """Apply the rotary encoding to every valid row (preproc.py:187-199).

    ``s``: (T, d) or (B, T, d) CUDA tensor (fp32 or bf16); ``timestamps``:
    None or (T,) / (B, T) event times (seconds; cast to fp64); ``lengths``:
    optional (B,) valid-row counts (rows 0..len-1 are the sequence, as the
    reference's unpadded (len, d) input)."""
    single = s.dim() == 2
    x = s.unsqueeze(0) if single else s
    if x.dim() != 3:
        raise ShapeError(f"rote_sequence expects (T, d) or (B, T, d), got {tuple(s.shape)}")
    if x.shape[-1] != 2 * cfg.half_dim:
        raise ShapeError(f"rotary config covers dim {2 * cfg.half_dim}, input has {x.shape[-1]}")
    _capi._need_cuda(x)
    x = x.contiguous()
    ts = None
    if timestamps is not None:
        ts = torch.as_tensor(timestamps, dtype=torch.float64, device=x.device).reshape(x.shape[0], x.shape[1])
        ts = ts.contiguous()
    ln = None
    if lengths is not None:
        ln = torch.as_tensor(lengths, device=x.device).to(torch.int32).contiguous()
        if ln.numel() != x.shape[0]:
            raise ShapeError(f"need one length per sample ({x.shape[0]}), got {ln.numel()}")
        if not torch.cuda.is_current_stream_capturing():  # (the kernels also clamp to [0, T])
            lo, hi = int(ln.min()), int(ln.max())
            if lo < 0 or hi > x.shape[1]:
                raise ValueError(f"lengths must lie in [0, {x.shape[1]}], got [{lo}, {hi}]")
    if x.numel() == 0:  # T = 0: the reference returns the (empty) input
        return s
    y = _Rote.apply(x, ln, ts, cfg)
    return y[0] if single else y


# ---------------------------------------------------------------------------
# Schemas (preproc.py:23-63, same validation messages)


@dataclass
class EventSchema:
    name: str
    vocab_size: int
    max_len: int

    def __post_init__(self):
        if self.vocab_size < 1:
            raise ValueError(f"event {self.name!r}: vocab size must be >= 1")
        if self.max_len < 1:
            raise ValueError(f"event {self.name!r}: max length must be >= 1")


@dataclass
class FeatureSchema:
    """Input layout: m dense values, n sparse ids, K event streams, dim d."""

    num_dense: int
    sparse_vocab_sizes: list
    events: list
    dim: int

    def __post_init__(self):
        if self.num_dense < 0:
            raise ValueError("dense feature count must be >= 0")
        for i, v in enumerate(self.sparse_vocab_sizes):
            if v < 1:
                raise ValueError(f"sparse feature {i}: vocab size must be >= 1")
        if self.dim < 2 or self.dim % 2 != 0:
            raise ValueError("embedding dim must be even and >= 2 (rotary pairs)")
        names = [e.name for e in self.events]
        if len(set(names)) != len(names):
            raise ValueError("event names must be unique")

    @property
    def num_sparse(self) -> int:
        return len(self.sparse_vocab_sizes)

    @property
    def num_tokens(self) -> int:
        """Rows of the assembled non-sequence matrix: dense block + n sparse."""
        return self.num_sparse + 1


# ---------------------------------------------------------------------------
# Non-sequence embedding


def _as_dev(x, like_device, dtype=None):
    t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x))
    return t.to(device=like_device, dtype=dtype or t.dtype)


def embed_dense(x_dense, proj):
    """Project the m raw dense values to one d-dim row (preproc.py:103-108):
    ``x_dense`` (m,) or (B, m); ``proj`` a (d, m) CUDA tensor or PRef."""
    shape = proj.w().shape if isinstance(proj, F.PRef) else proj.shape
    dev = proj.P.device if isinstance(proj, F.PRef) else proj.device
    dt = proj.P.compute_dtype if isinstance(proj, F.PRef) else proj.dtype
    x = _as_dev(x_dense, dev, dt)
    single = x.dim() == 1
    if x.dim() not in (1, 2) or x.shape[-1] != shape[1]:
        raise ShapeError(f"dense projection {tuple(shape)} does not accept input of shape {tuple(x.shape)}")
    pt = F.PRef(proj.P, proj.key, lambda w: w.t()) if isinstance(proj, F.PRef) else proj.t()
    y = F.mm(x.reshape(-1, shape[1]), pt)
    return y[0] if single else y


def embed_sparse(index, table):
    """Row lookup = one-hot product with the table (preproc.py:111-116);
    ``index`` an int or a (B,) integer array, ``table`` a (V, d) CUDA tensor.
    IndexError outside the vocabulary (checked on the host)."""
    idx = np.asarray(index).astype(np.int64)
    V = table.shape[0]
    if idx.size and (idx.min() < 0 or idx.max() >= V):
        bad = int(idx.min()) if idx.min() < 0 else int(idx.max())
        raise IndexError(f"sparse id {bad} outside vocab of size {V}")
    rows = table[torch.as_tensor(idx, device=table.device)]
    return rows


def assemble_nonseq(dense_emb, sparse_embs):
    """Stack dense-first into the (n+1, d) — batched (B, n+1, d) —
    non-sequence matrix (preproc.py:119-127)."""
    d = dense_emb.shape[-1]
    for i, e in enumerate(sparse_embs):
        if e.shape != dense_emb.shape:
            raise ShapeError(f"sparse embedding {i} has shape {tuple(e.shape)}, expected {tuple(dense_emb.shape)} "
                             f"(d = {d})")
    return torch.stack([dense_emb] + list(sparse_embs), dim=-2)


@dataclass
class NonSeqEmbeddingParams:
    """Dense projection ``{prefix}/dense_proj`` (d, m) and the sparse tables
    ``{prefix}/sparse{i}`` (vocab_i, d), stacked in one block so a single
    gather kernel serves every feature (embed_nonseq)."""

    P: Params
    prefix: str
    schema: FeatureSchema
    offsets: np.ndarray

    @property
    def proj(self):
        return f"{self.prefix}/dense_proj"

    @property
    def tables(self):
        return f"{self.prefix}#tables"

    @classmethod
    def create(cls, params: Params, prefix: str, schema: FeatureSchema,
               rng: np.random.Generator | None = None) -> "NonSeqEmbeddingParams":
        rng = rng if rng is not None else np.random.default_rng(0)
        d, m = schema.dim, schema.num_dense
        sizes = list(schema.sparse_vocab_sizes)
        offsets = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
        p = cls(params, prefix, schema, offsets)
        params.add(p.proj, rng.normal(0.0, 1.0 / np.sqrt(max(m, 1)), (d, m)))
        params.block(p.tables, (int(offsets[-1]), d))
        for i, v in enumerate(sizes):
            params.add(f"{prefix}/sparse{i}", rng.normal(0.0, 1.0 / np.sqrt(d), (v, d)), block=p.tables,
                       index=slice(int(offsets[i]), int(offsets[i + 1])))
        return p


class _EmbedNonseq(torch.autograd.Function):
    """kl_embed_nonseq_fwd / _bwd: embed_dense + embed_sparse + assemble_nonseq
    in one gather pass; the VJP scatter-adds into the tables' gradient rows
    and accumulates the projection gradient (both in Params.gflat)."""

    @staticmethod
    def forward(ctx, flat, p, x_dense, ids, offsets):
        P = p.P
        B, n = ids.shape
        d, m = p.schema.dim, p.schema.num_dense
        table, proj = P.w(p.tables), P.w(p.proj)
        out = torch.empty(B, n + 1, d, device=table.device, dtype=table.dtype)
        _capi.call("kl_embed_nonseq_fwd", B, n, d, m, _capi.dt(table), x_dense.data_ptr(), proj.data_ptr(),
                   table.data_ptr(), offsets.data_ptr(), ids.data_ptr(), int(table.shape[0]), out.data_ptr(),
                   _capi._stream())
        ctx.p, ctx.B, ctx.n = p, B, n
        ctx.save_for_backward(x_dense, ids, offsets)
        return out

    @staticmethod
    def backward(ctx, g):
        x_dense, ids, offsets = ctx.saved_tensors
        p = ctx.p
        P = p.P
        g = g.contiguous()
        gt = P.g(p.tables)
        _capi.call("kl_embed_nonseq_bwd", ctx.B, ctx.n, p.schema.dim, p.schema.num_dense, _capi.dt(g),
                   x_dense.data_ptr(), g.data_ptr(), offsets.data_ptr(), ids.data_ptr(), int(gt.shape[0]),
                   gt.data_ptr(), P.g(p.proj).data_ptr(), _capi._stream())
        return None, None, None, None, None


def embed_nonseq(x_dense, sparse_ids, p: NonSeqEmbeddingParams, check_ids: bool = True) -> torch.Tensor:
    """The assembled non-sequence matrix (B, n+1, d) = [embed_dense(x) |
    embed_sparse(id_i, table_i) ...] (preproc.py:103-127) in ONE kernel.
    ``x_dense`` (B, m) float, ``sparse_ids`` (B, n) integers; ids outside a
    feature's vocabulary raise IndexError (checked on the host unless
    ``check_ids`` is False, e.g. inside CUDA-graph capture)."""
    P = p.P
    dev = P.device
    xd = _as_dev(x_dense, dev, torch.float32).contiguous()
    ids = _as_dev(sparse_ids, dev, torch.int64).contiguous()
    n = p.schema.num_sparse
    if xd.dim() != 2 or xd.shape[1] != p.schema.num_dense or ids.shape != (xd.shape[0], n):
        raise ShapeError(f"need x_dense (B, {p.schema.num_dense}) and sparse ids (B, {n}), got "
                         f"{tuple(xd.shape)} / {tuple(ids.shape)}")
    if check_ids and n and not torch.cuda.is_current_stream_capturing():
        lo = ids.min(0).values.cpu().numpy()
        hi = ids.max(0).values.cpu().numpy()
        for i, v in enumerate(p.schema.sparse_vocab_sizes):
            if lo[i] < 0 or hi[i] >= v:
                bad = int(lo[i]) if lo[i] < 0 else int(hi[i])
                raise IndexError(f"sparse id {bad} outside vocab of size {v}")
    offsets = torch.as_tensor(p.offsets[:-1], device=dev, dtype=torch.int64)
    return _EmbedNonseq.apply(P.flat, p, xd, ids, offsets)


def fuse_sequences(seqs, fusion):
    """Rowwise MLP over the (T, K*d) — batched (B, T, K*d) — concatenation
    of K aligned sequences (preproc.py:130-143)."""
    if not seqs:
        raise ShapeError("fusion needs at least one sequence")
    t = seqs[0].shape[-2]
    for s in seqs:
        if s.shape[-2] != t or s.dim() != seqs[0].dim():
            raise ShapeError("sequences must share length T before fusion")
    cat = seqs[0] if len(seqs) == 1 else torch.cat(list(seqs), dim=-1)
    if fusion.in_dim != cat.shape[-1]:
        raise ShapeError(f"fusion expects width {fusion.in_dim}, got {cat.shape[-1]}")
    if t == 0:
        return cat.new_zeros(cat.shape[:-1] + (fusion.out_dim,))
    return fusion.apply_rows(cat)


def align_right(seqs, target_len: int):
    """Zero-pad each (T_i, d) sequence at the front so the newest rows align
    (preproc.py:146-152); numpy arrays or tensors, returned in kind."""
    out = []
    for s in seqs:
        pad = target_len - s.shape[0]
        if pad < 0:
            raise ShapeError(f"sequence of length {s.shape[0]} exceeds target {target_len}")
        if isinstance(s, torch.Tensor):
            out.append(torch.cat([s.new_zeros(pad, s.shape[1]), s], dim=0) if pad else s)
        else:
            out.append(np.concatenate([np.zeros((pad, s.shape[1])), s], axis=0) if pad else s)
    return out
