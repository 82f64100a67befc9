"""Synthetic CTR batches of a named config (SPEC.md:628-646 generator
contract, reduced to what the layer hot path consumes): non-sequence tokens
X ~ N(0, 1/d) (embedding init scale), per-event sequences
S_e ~ N(0, 1/d) with lengths, labels ~ Bernoulli(p) with a ground-truth
click probability p in (0.02, 0.5).  Deterministic given the seed."""

from __future__ import annotations

import numpy as np


def ctr_batch(cfg, B: int, seed: int = 0, full_length: bool = True, dtype=np.float32):
    rng = np.random.default_rng(seed)
    d = cfg.d
    X = rng.normal(0.0, 1.0 / np.sqrt(d), (B, cfg.n_ctx, d)).astype(dtype)
    S, lengths = [], []
    for ev in cfg.events:
        S.append(rng.normal(0.0, 1.0 / np.sqrt(d), (B, ev.T, d)).astype(dtype))
        if full_length:
            lengths.append(np.full(B, ev.T, dtype=np.int32))
        else:
            lengths.append(rng.integers(0, ev.T + 1, size=B).astype(np.int32))
    # ground truth: a fixed random probe of the context tokens and of the
    # most recent behaviour rows, squashed into CTR (0.02, 0.5)
    probe = rng.normal(0.0, 1.0, d)
    z = X.mean(axis=1) @ probe * np.sqrt(d)
    for e, s in enumerate(S):
        last = s[np.arange(B), np.maximum(lengths[e] - 1, 0)]
        z = z + last @ probe * np.sqrt(d) * 0.5
    p = 0.02 + 0.48 / (1.0 + np.exp(-z))
    labels = (rng.random(B) < p).astype(np.float32)
    return X, S, lengths, labels
