"""Primitive float64 ops with explicit VJPs (oracle; test infrastructure only).

Each function returns ``(out, bwd)`` where ``bwd(g)`` returns the gradients of
the inputs that carry them.  Restated from /root/reference/pkg/src/kunlun/
tensor.py; the cited lines are the reference semantics being reproduced.
"""

from __future__ import annotations

import numpy as np

# Activation tags in the reference's table order (tensor.py:431-440).  The
# integer codes are the ones the C-ABI uses (include/kunlun_capi.h).
ACT_CODES = {
    "identity": 0,
    "relu": 1,
    "silu": 2,
    "tanh": 3,
    "sigmoid": 4,
    "exp": 5,
    "sqrt": 6,
    "log": 7,
}


def sigmoid(x: np.ndarray) -> np.ndarray:
    """Stable logistic (tensor.py:403-409)."""
    x = np.asarray(x, dtype=np.float64)
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def act_fwd(kind: str, x: np.ndarray) -> np.ndarray:
    """Forward of the activation table (tensor.py:431-440)."""
    if kind == "identity":
        return x.copy()
    if kind == "relu":
        return np.maximum(x, 0.0)
    if kind == "silu":
        return x * sigmoid(x)
    if kind == "tanh":
        return np.tanh(x)
    if kind == "sigmoid":
        return sigmoid(x)
    if kind == "exp":
        return np.exp(x)
    if kind == "sqrt":
        return np.sqrt(x)
    if kind == "log":
        return np.log(x)
    raise ValueError(f"unknown activation {kind!r}")


def act_dfn(kind: str, x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """Derivative dfn(x, y) of the activation table (tensor.py:425-440).

    relu'(0) = 0 (tensor.py:433); silu' = s(1 + x(1 - s)) (tensor.py:425-427).
    """
    if kind == "identity":
        return np.ones_like(x)
    if kind == "relu":
        return (x > 0).astype(np.float64)
    if kind == "silu":
        s = sigmoid(x)
        return s * (1.0 + x * (1.0 - s))
    if kind == "tanh":
        return 1.0 - y * y
    if kind == "sigmoid":
        return y * (1.0 - y)
    if kind == "exp":
        return y.copy()
    if kind == "sqrt":
        return 0.5 / y
    if kind == "log":
        return 1.0 / x
    raise ValueError(f"unknown activation {kind!r}")


def masked_softmax(a: np.ndarray, mask: np.ndarray):
    """Softmax over the last axis restricted to ``mask``; fully-masked rows
    give 0 (tensor.py:485-505).  VJP y*(g - sum(g*y)) (tensor.py:501-503)."""
    m = np.broadcast_to(mask, a.shape)
    neg = np.where(m, a, -np.inf)
    if a.shape[-1]:
        rowmax = neg.max(axis=-1, keepdims=True)
    else:
        rowmax = np.zeros(a.shape[:-1] + (1,))
    rowmax = np.where(np.isfinite(rowmax), rowmax, 0.0)
    e = np.exp(np.where(m, a - rowmax, -np.inf))
    denom = e.sum(axis=-1, keepdims=True)
    y = np.divide(e, denom, out=np.zeros_like(e), where=denom > 0)

    def bwd(g):
        inner = (g * y).sum(axis=-1, keepdims=True)
        return y * (g - inner)

    return y, bwd


def rms_norm(x: np.ndarray, gain: np.ndarray, eps: float = 1e-6):
    """x / sqrt(mean(x^2) + eps) * gain, eps inside the sqrt (tensor.py:552-556)."""
    d = x.shape[-1]
    ms = (x * x).mean(axis=-1, keepdims=True)
    s = 1.0 / np.sqrt(ms + eps)
    xn = x * s
    y = xn * gain

    def bwd(g):
        gg = g * gain
        dx = s * gg - (s ** 3) / d * x * (gg * x).sum(axis=-1, keepdims=True)
        dgain = (g * xn).reshape(-1, d).sum(axis=0)
        return dx, dgain

    return y, bwd


def bce_with_logits(z: np.ndarray, y: np.ndarray):
    """Mean BCE in nats, stable for large |z| (tensor.py:535-549)."""
    z = np.asarray(z, dtype=np.float64)
    y = np.asarray(y, dtype=np.float64)
    n = max(z.size, 1)
    loss = float((np.maximum(z, 0.0) - y * z + np.log1p(np.exp(-np.abs(z)))).sum() / n)

    def bwd(g=1.0):
        return (sigmoid(z) - y) * (float(g) / n)

    return loss, bwd


def normalized_entropy(labels, preds, from_logits: bool = False) -> dict:
    """NE = cross entropy / background entropy (PAPER.md:438-446 Eq. A1-A2;
    SPEC.md:540-561 ``normalized_entropy`` / ``NeReport``), natural log, float64.
    Probabilities are clipped to [1e-12, 1 - 1e-12]; logits use
    the stable log-sigmoid.  All-zero / all-one labels raise."""
    y = np.asarray(labels, dtype=np.float64).ravel()
    p = np.asarray(preds, dtype=np.float64).ravel()
    if y.size < 1 or y.size != p.size:
        raise ValueError("normalized_entropy: need N >= 1 labels and predictions")
    if from_logits:
        lp = -np.log1p(np.exp(-np.abs(p))) + np.minimum(p, 0.0)
        lq = -np.log1p(np.exp(-np.abs(p))) - np.maximum(p, 0.0)
    else:
        c = np.clip(p, 1e-12, 1.0 - 1e-12)
        lp, lq = np.log(c), np.log1p(-c)
    ce = float(-(y * lp + (1.0 - y) * lq).mean())
    ctr = float(y.mean())
    if not 0.0 < ctr < 1.0:
        raise ValueError("degenerate background entropy")
    h = float(-ctr * np.log(ctr) - (1.0 - ctr) * np.log1p(-ctr))
    return {"cross_entropy": ce, "background_entropy": h, "ne": ce / h, "ctr": ctr, "n": int(y.size)}


def rote_angles(t_len: int, timestamps, pos_freqs, temp_freqs, tau_scale: float, gap_mode: str) -> np.ndarray:
    """(T, d/2) rotation angles of rote_sequence (preproc.py:187-199): row
    position t times pos_freqs plus tau = log1p(max(gap, 0) / tau_scale) times
    temp_freqs; gaps to the previous event or below the newest
    (gaps_from_timestamps, preproc.py:175-184); no timestamps -> tau = 0."""
    pos = np.arange(t_len, dtype=np.float64)
    if timestamps is None or t_len == 0:
        taus = np.zeros(t_len)
    else:
        ts = np.asarray(timestamps, dtype=np.float64)
        gaps = np.concatenate([[0.0], np.diff(ts)]) if gap_mode == "previous" else ts[-1] - ts
        taus = np.log1p(np.maximum(gaps, 0.0) / tau_scale)
    return pos[:, None] * np.asarray(pos_freqs)[None, :] + taus[:, None] * np.asarray(temp_freqs)[None, :]


def rotate_pairs(x: np.ndarray, ang: np.ndarray):
    """Per-plane rotation of (even, odd) pairs (tensor.py:508-532); the VJP
    rotates the cotangent by the negative angles."""
    x = np.asarray(x, dtype=np.float64)
    c, s = np.cos(ang), np.sin(ang)
    y = np.empty_like(x)
    y[..., 0::2] = x[..., 0::2] * c - x[..., 1::2] * s
    y[..., 1::2] = x[..., 0::2] * s + x[..., 1::2] * c

    def bwd(g):
        g = np.asarray(g, dtype=np.float64)
        gx = np.empty_like(g)
        gx[..., 0::2] = g[..., 0::2] * c + g[..., 1::2] * s
        gx[..., 1::2] = -g[..., 0::2] * s + g[..., 1::2] * c
        return gx

    return y, bwd


def rote_sequence(x: np.ndarray, timestamps, pos_freqs, temp_freqs, tau_scale: float = 60.0,
                  gap_mode: str = "previous"):
    """ROTE on a (T, d) sequence (preproc.py:187-199)."""
    x = np.asarray(x, dtype=np.float64)
    return rotate_pairs(x, rote_angles(x.shape[0], timestamps, pos_freqs, temp_freqs, tau_scale, gap_mode))


def mlp_rows(x: np.ndarray, ws, bs, acts):
    """Rowwise (linear, bias, act) stack; "identity" skips the act (mlp.py:47-54)."""
    caches = []
    h = x
    for w, b, act in zip(ws, bs, acts):
        pre = h @ w.T + b
        post = pre if act == "identity" else act_fwd(act, pre)
        caches.append((h, pre, post))
        h = post

    def bwd(g):
        dws, dbs = [None] * len(ws), [None] * len(ws)
        for i in reversed(range(len(ws))):
            hin, pre, post = caches[i]
            if acts[i] != "identity":
                g = g * act_dfn(acts[i], pre, post)
            dws[i] = g.reshape(-1, g.shape[-1]).T @ hin.reshape(-1, hin.shape[-1])
            dbs[i] = g.reshape(-1, g.shape[-1]).sum(axis=0)
            g = g @ ws[i]
        return g, dws, dbs

    return h, bwd


# ---------------------------------------------------------------------------
# preproc.py:103-152 — raw features to embeddings


def embed_nonseq(x_dense, ids, proj, tables):
    """[proj x | table_0[id_0] | ...] (embed_dense preproc.py:103-108 as a
    matvec, embed_sparse 111-116 as a row lookup, assemble_nonseq 119-127).
    Returns (out (n+1, d), bwd(g) -> (dproj, [dtable_i]))."""
    rows = [proj @ x_dense] + [t[int(i)] for t, i in zip(tables, ids)]
    out = np.stack(rows)

    def bwd(g):
        dproj = np.outer(g[0], x_dense)
        dts = []
        for k, (t, i) in enumerate(zip(tables, ids)):
            dt = np.zeros_like(t)
            dt[int(i)] += g[1 + k]
            dts.append(dt)
        return dproj, dts

    return out, bwd


def align_right(seqs, target_len: int):
    """preproc.py:146-152."""
    out = []
    for s in seqs:
        pad = target_len - s.shape[0]
        if pad < 0:
            raise ValueError(f"sequence of length {s.shape[0]} exceeds target {target_len}")
        out.append(np.concatenate([np.zeros((pad, s.shape[1])), s], axis=0) if pad else s)
    return out


def fuse_sequences(seqs, ws, bs, acts):
    """Rowwise MLP over the (T, K*d) concatenation (preproc.py:130-143)."""
    cat = np.concatenate(seqs, axis=1)
    y, mbwd = mlp_rows(cat, ws, bs, acts)

    def bwd(g):
        dcat, dws, dbs = mbwd(g)
        widths = np.cumsum([0] + [s.shape[1] for s in seqs])
        return [dcat[:, a:b] for a, b in zip(widths[:-1], widths[1:])], dws, dbs

    return y, bwd
