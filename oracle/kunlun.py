"""Per-sample float64 restatement of the Kunlun hot-path modules (oracle;
test infrastructure only).

Parameters live in a flat ``dict[name -> ndarray]`` keyed by the reference's
registry names (gdpa.py:89-92, attention.py:42-45, seqsum.py:62-77/177-183,
interaction.py:93-98/137-140, mlp.py:31-33).  Each op returns ``(out, bwd)``;
``bwd(g)`` returns input gradients plus a ``dict`` of parameter gradients.
Formulations follow the reference code line by line (no reassociation), so
this is an independent check of the reassociated GPU kernels.
"""

from __future__ import annotations

from collections import defaultdict

import numpy as np

from .ops import act_dfn, act_fwd, masked_softmax, mlp_rows, rms_norm

DEFAULT_ACTIVATION_CYCLE = ("silu", "relu", "identity", "tanh")  # gdpa.py:31


def _acc(dst: dict, name: str, g: np.ndarray) -> None:
    if name in dst:
        dst[name] = dst[name] + g
    else:
        dst[name] = g


def heads_of(p: dict, prefix: str) -> int:
    h = 0
    while f"{prefix}/head{h}/w_q" in p:
        h += 1
    return h


# ---------------------------------------------------------------------------
# attention.py
# ---------------------------------------------------------------------------


def band_mask(t_len: int, w: int, causal: bool = False) -> np.ndarray:
    """|i-j| <= w (and j <= i if causal) (attention.py:96-103)."""
    idx = np.arange(t_len)
    diff = idx[None, :] - idx[:, None]
    m = np.abs(diff) <= w
    if causal:
        m &= diff <= 0
    return m


def band_support_sizes(t_len: int, w: int, causal: bool = False) -> np.ndarray:
    """Per-query key count (attention.py:132-139)."""
    idx = np.arange(t_len)
    hi = np.minimum(idx + w, t_len - 1)
    lo = np.maximum(idx - w, 0)
    if causal:
        hi = idx
    return hi - lo + 1


def length_mask(t_len: int, length) -> np.ndarray:
    """attention.py:106-112."""
    valid = np.ones(t_len, dtype=bool)
    if length is not None:
        if not 0 <= length <= t_len:
            raise ValueError(f"valid length {length} outside [0, {t_len}]")
        valid[length:] = False
    return valid


def multi_head_attention(xq, xkv, p: dict, prefix: str, mask=None):
    """softmax(mask, (xWq^T)(yWk^T)^T / sqrt(d_h)) (yWv^T), concat, W_out^T;
    no residual; fully-masked rows -> 0 (attention.py:69-93)."""
    H = heads_of(p, prefix)
    Wq = np.stack([p[f"{prefix}/head{h}/w_q"] for h in range(H)])  # (H,dh,d)
    Wk = np.stack([p[f"{prefix}/head{h}/w_k"] for h in range(H)])
    Wv = np.stack([p[f"{prefix}/head{h}/w_v"] for h in range(H)])
    Wo = p[f"{prefix}/w_out"]
    n_q, n_k = xq.shape[0], xkv.shape[0]
    d_h = Wq.shape[1]
    if mask is None:
        mask = np.ones((n_q, n_k), dtype=bool)
    inv = 1.0 / np.sqrt(d_h)
    q = xq @ Wq.transpose(0, 2, 1)  # (H, n, d_h); batched BLAS, same sums as the einsum
    k = xkv @ Wk.transpose(0, 2, 1)
    v = xkv @ Wv.transpose(0, 2, 1)
    scores = (q @ k.transpose(0, 2, 1)) * inv
    attn, sm_bwd = masked_softmax(scores, mask[None])
    o = attn @ v
    cat = o.transpose(1, 0, 2).reshape(n_q, H * d_h)
    out = cat @ Wo.T

    def bwd(g):
        grads = {}
        grads[f"{prefix}/w_out"] = g.T @ cat
        dcat = g @ Wo
        do = dcat.reshape(n_q, H, d_h).transpose(1, 0, 2)
        dattn = do @ v.transpose(0, 2, 1)
        dv = attn.transpose(0, 2, 1) @ do
        dscores = sm_bwd(dattn) * inv
        dq = dscores @ k
        dk = dscores.transpose(0, 2, 1) @ q
        dWq = dq.transpose(0, 2, 1) @ xq
        dWk = dk.transpose(0, 2, 1) @ xkv
        dWv = dv.transpose(0, 2, 1) @ xkv
        for h in range(H):
            grads[f"{prefix}/head{h}/w_q"] = dWq[h]
            grads[f"{prefix}/head{h}/w_k"] = dWk[h]
            grads[f"{prefix}/head{h}/w_v"] = dWv[h]
        dxq = (dq @ Wq).sum(0)
        dxkv = (dk @ Wk).sum(0) + (dv @ Wv).sum(0)
        return dxq, dxkv, grads

    return out, bwd


BAND_MIN_T = 1024  # mha_window evaluates block-banded above this length (same sums, no T x T arrays)
BAND_BLOCK = 128


def _banded_self_attention(x, p: dict, prefix: str, w: int, causal: bool, valid):
    """multi_head_attention(x, x, p, prefix, band & valid) evaluated per
    128-query block over the key rows that block can see ([q0 - w, q0 + 127 +
    w]): every score outside that range is masked in the reference
    (attention.py:69-93 with band_mask, attention.py:96-104), so it contributes
    an exact zero to the masked softmax (tensor.py:485-505) and to every
    product — the result equals the dense evaluation up to float64 summation
    order (tests/test_oracle_golden.py checks them against each other)."""
    H = heads_of(p, prefix)
    Wq = np.stack([p[f"{prefix}/head{h}/w_q"] for h in range(H)])
    Wk = np.stack([p[f"{prefix}/head{h}/w_k"] for h in range(H)])
    Wv = np.stack([p[f"{prefix}/head{h}/w_v"] for h in range(H)])
    Wo = p[f"{prefix}/w_out"]
    T = x.shape[0]
    d_h = Wq.shape[1]
    inv = 1.0 / np.sqrt(d_h)
    q = x @ Wq.transpose(0, 2, 1)
    k = x @ Wk.transpose(0, 2, 1)
    v = x @ Wv.transpose(0, 2, 1)
    o = np.zeros((H, T, d_h))
    blocks = []
    for q0 in range(0, T, BAND_BLOCK):
        q1 = min(T, q0 + BAND_BLOCK)
        k0, k1 = max(0, q0 - w), min(T, q1 + w)
        qi = np.arange(q0, q1)[:, None]
        kj = np.arange(k0, k1)[None, :]
        m = (np.abs(qi - kj) <= w) & valid[q0:q1, None] & valid[None, k0:k1]
        if causal:
            m &= kj <= qi
        sc = (q[:, q0:q1] @ k[:, k0:k1].transpose(0, 2, 1)) * inv
        attn, sm_bwd = masked_softmax(sc, m[None])
        o[:, q0:q1] = attn @ v[:, k0:k1]
        blocks.append((q0, q1, k0, k1, attn, sm_bwd))
    cat = o.transpose(1, 0, 2).reshape(T, H * d_h)
    out = cat @ Wo.T

    def bwd(g):
        grads = {f"{prefix}/w_out": g.T @ cat}
        do = (g @ Wo).reshape(T, H, d_h).transpose(1, 0, 2)
        dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
        for q0, q1, k0, k1, attn, sm_bwd in blocks:
            dattn = do[:, q0:q1] @ v[:, k0:k1].transpose(0, 2, 1)
            dv[:, k0:k1] += attn.transpose(0, 2, 1) @ do[:, q0:q1]
            dsc = sm_bwd(dattn) * inv
            dq[:, q0:q1] += dsc @ k[:, k0:k1]
            dk[:, k0:k1] += dsc.transpose(0, 2, 1) @ q[:, q0:q1]
        dWq, dWk, dWv = dq.transpose(0, 2, 1) @ x, dk.transpose(0, 2, 1) @ x, dv.transpose(0, 2, 1) @ x
        for h in range(H):
            grads[f"{prefix}/head{h}/w_q"] = dWq[h]
            grads[f"{prefix}/head{h}/w_k"] = dWk[h]
            grads[f"{prefix}/head{h}/w_v"] = dWv[h]
        dx = (dq @ Wq).sum(0) + (dk @ Wk).sum(0) + (dv @ Wv).sum(0)
        return dx, np.zeros_like(x), grads

    return out, bwd


def mha_window(s, p: dict, prefix: str, w: int, causal: bool = False, length=None, banded=None):
    """S + MHA(S, S, band & valid) (attention.py:124-129).  ``banded``
    (default: T > BAND_MIN_T) evaluates the same masked attention per query
    block over its visible key range (_banded_self_attention)."""
    t_len = s.shape[0]
    valid = length_mask(t_len, length)
    if banded is None:
        banded = t_len > BAND_MIN_T
    if banded:
        a, a_bwd = _banded_self_attention(s, p, prefix, w, causal, valid)
    else:
        mask = band_mask(t_len, w, causal) & valid[None, :] & valid[:, None]
        a, a_bwd = multi_head_attention(s, s, p, prefix, mask)

    def bwd(g):
        dxq, dxkv, grads = a_bwd(g)
        return g + dxq + dxkv, grads

    return a + s, bwd


def mha_full(s, p: dict, prefix: str, length=None):
    """attention.py:115-121."""
    t_len = s.shape[0]
    valid = length_mask(t_len, length)
    mask = valid[None, :] & valid[:, None]
    a, a_bwd = multi_head_attention(s, s, p, prefix, mask)

    def bwd(g):
        dxq, dxkv, grads = a_bwd(g)
        return g + dxq + dxkv, grads

    return a + s, bwd


# ---------------------------------------------------------------------------
# gdpa.py
# ---------------------------------------------------------------------------


def summarize_nonseq(x, pool):
    """X_sum = P X (gdpa.py:96-100)."""
    out = pool @ x

    def bwd(g):
        return pool.T @ g, g @ x.T  # dx, dpool

    return out, bwd


def generate_kv(x_sum, p: dict, prefix: str, n_kv: int):
    """Per head K_h = reshape(KG_h flat, (n_kv, d_h)), same for V (gdpa.py:103-112)."""
    H = heads_of(p, prefix)
    flat = x_sum.reshape(-1)
    kvs = []
    for h in range(H):
        kg = p[f"{prefix}/head{h}/w_kgen"]
        vg = p[f"{prefix}/head{h}/w_vgen"]
        d_h = kg.shape[0] // n_kv
        kvs.append(((kg @ flat).reshape(n_kv, d_h), (vg @ flat).reshape(n_kv, d_h)))

    def bwd(dkvs):
        grads = {}
        dflat = np.zeros_like(flat)
        for h, (dk, dv) in enumerate(dkvs):
            kg = p[f"{prefix}/head{h}/w_kgen"]
            vg = p[f"{prefix}/head{h}/w_vgen"]
            grads[f"{prefix}/head{h}/w_kgen"] = np.outer(dk.reshape(-1), flat)
            grads[f"{prefix}/head{h}/w_vgen"] = np.outer(dv.reshape(-1), flat)
            dflat = dflat + kg.T @ dk.reshape(-1) + vg.T @ dv.reshape(-1)
        return dflat.reshape(x_sum.shape), grads

    return kvs, bwd


def gdpa_forward(s, kvs, p: dict, prefix: str, tau: float, acts):
    """Y = concat_h Act_h(Q_h K_h^T / tau) V_h  W_out^T + S with Q_h = S Wq_h^T
    (gdpa.py:120-138; blockwise gdpa.py:190-206 is equal to <=1e-10).
    Returns dS and dK/dV per head so the caller can chain generate_kv."""
    H = len(kvs)
    inv_tau = 1.0 / tau
    Wo = p[f"{prefix}/w_out"]
    cache = []
    outs = []
    for h, (k, v) in enumerate(kvs):
        wq = p[f"{prefix}/head{h}/w_q"]
        q = s @ wq.T
        z = (q @ k.T) * inv_tau
        a = act_fwd(acts[h], z)
        outs.append(a @ v)
        cache.append((wq, q, z, a, k, v))
    cat = np.concatenate(outs, axis=1)
    y = cat @ Wo.T + s

    def bwd(g):
        grads = {f"{prefix}/w_out": g.T @ cat}
        dcat = g @ Wo
        ds = g.copy()
        dkvs = []
        d_h = cache[0][0].shape[0]
        for h in range(H):
            wq, q, z, a, k, v = cache[h]
            do = dcat[:, h * d_h:(h + 1) * d_h]
            dv = a.T @ do
            da = do @ v.T
            dz = da * act_dfn(acts[h], z, a) * inv_tau
            dq = dz @ k
            dk = dz.T @ q
            grads[f"{prefix}/head{h}/w_q"] = dq.T @ s
            ds = ds + dq @ wq
            dkvs.append((dk, dv))
        return ds, dkvs, grads

    return y, bwd


# ---------------------------------------------------------------------------
# seqsum.py
# ---------------------------------------------------------------------------


def split_for_budget(budget: int):
    """(b//4, b - 2(b//4), b//4) (seqsum.py:141-145)."""
    n_cls = budget // 4
    n_recent = budget // 4
    return n_cls, budget - n_cls - n_recent, n_recent


def hsp_init_bounds(n_seeds: int, n_tokens: int) -> np.ndarray:
    """Seed->token block bounds used by HspParams.create (seqsum.py:67-71)."""
    return np.linspace(0, n_seeds, n_tokens + 1).astype(int)


def sumkronlinear(x, zs, ws):
    """Y = sum_i Z_i^T X W_i (seqsum.py:105-122)."""
    y = sum(z.T @ x @ w for z, w in zip(zs, ws))

    def bwd(g):
        dx = np.zeros_like(x)
        dzs, dws = [], []
        for z, w in zip(zs, ws):
            zx = z.T @ x
            dws.append(zx.T @ g)
            gw = g @ w.T          # d(Z^T X)
            dzs.append(x @ gw.T)  # (S,D)(D,T) -> (S,T)
            dx = dx + z @ gw
        return dx, dzs, dws

    return y, bwd


def recent_rows(s, n_recent: int):
    """Last n_recent rows, front zero-padded (seqsum.py:186-196)."""
    t_len, d = s.shape
    out = np.zeros((n_recent, d))
    take = min(n_recent, t_len)
    if take > 0:
        out[n_recent - take:] = s[t_len - take:]

    def bwd(g):
        ds = np.zeros_like(s)
        if take > 0:
            ds[t_len - take:] += g[n_recent - take:]
        return ds

    return out, bwd


def hsp_summarize(s, p: dict, prefix: str, budget: int):
    """[CLS | SumKron(seed-attend) | recent] (seqsum.py:199-210; pma 26-34;
    hsp_seed_attend 96-102).  Empty sequences give constant zeros (no grad)."""
    n_cls, n_tok, n_rec = split_for_budget(budget)
    d = s.shape[1]
    t_len = s.shape[0]
    grads_acc = {}
    parts = []
    bwds = []
    if n_cls > 0:
        if t_len == 0:
            parts.append(np.zeros((n_cls, d)))
            bwds.append(None)
        else:
            qc = p[f"{prefix}/cls_queries"]
            c, c_bwd = multi_head_attention(qc, s, p, f"{prefix}/cls_attn")
            parts.append(c)
            bwds.append(("cls", c_bwd))
    rank = 0
    while f"{prefix}/hsp/kron{rank}/seq_map" in p:
        rank += 1
    zs = [p[f"{prefix}/hsp/kron{i}/seq_map"] for i in range(rank)]
    ws = [p[f"{prefix}/hsp/kron{i}/emb_map"] for i in range(rank)]
    seeds = p[f"{prefix}/hsp/seeds"]
    if t_len == 0:
        hseed = np.zeros(seeds.shape)
        hs_bwd = None
        n_bwd = None
    else:
        qn, n_bwd = rms_norm(seeds, p[f"{prefix}/hsp/norm_gain"])
        hseed, hs_bwd = multi_head_attention(qn, s, p, f"{prefix}/hsp/attn")
    htok, k_bwd = sumkronlinear(hseed, zs, ws)
    parts.append(htok)
    rec, r_bwd = recent_rows(s, n_rec)
    parts.append(rec)
    rows = np.concatenate(parts, axis=0) if parts else np.zeros((0, d))

    def bwd(g):
        grads = dict(grads_acc)
        ds = np.zeros_like(s)
        off = 0
        if n_cls > 0:
            gc = g[off:off + n_cls]
            off += n_cls
            if bwds[0] is not None:
                dq, dkv, gr = bwds[0][1](gc)
                ds = ds + dkv
                grads.update(gr)
                grads[f"{prefix}/cls_queries"] = dq
        gt = g[off:off + n_tok]
        off += n_tok
        dh, dzs, dws = k_bwd(gt)
        for i in range(rank):
            grads[f"{prefix}/hsp/kron{i}/seq_map"] = dzs[i]
            grads[f"{prefix}/hsp/kron{i}/emb_map"] = dws[i]
        if hs_bwd is not None:
            dqn, dkv, gr = hs_bwd(dh)
            grads.update(gr)
            ds = ds + dkv
            dseeds, dgain = n_bwd(dqn)
            grads[f"{prefix}/hsp/seeds"] = dseeds
            grads[f"{prefix}/hsp/norm_gain"] = dgain
        gr_ = g[off:off + n_rec]
        ds = ds + r_bwd(gr_)
        return ds, grads

    return rows, bwd


# ---------------------------------------------------------------------------
# interaction.py
# ---------------------------------------------------------------------------


def expert_ranges(total: int, num_experts: int):
    """Balanced contiguous split, earlier experts +1 (interaction.py:50-60)."""
    if num_experts < 1 or num_experts > total:
        raise ValueError(f"cannot split {total} tokens across {num_experts} experts")
    base, extra = divmod(total, num_experts)
    ranges, pos = [], 0
    for i in range(num_experts):
        size = base + (1 if i < extra else 0)
        ranges.append((pos, pos + size))
        pos += size
    return ranges


def wukong_expert(x, p: dict, prefix: str):
    """x + g_deep*MLP(x) + g_dot*reshape(DotMap triu(x x^T)) (interaction.py:106-121)."""
    n_i, d = x.shape
    rows, cols = np.triu_indices(n_i)
    gram = x @ x.T
    tri = gram[rows, cols]
    dm = p[f"{prefix}/dot_map"]
    dot_out = (dm @ tri).reshape(n_i, d)
    ws = [p[f"{prefix}/deep/w0"], p[f"{prefix}/deep/w1"]]
    bs = [p[f"{prefix}/deep/b0"], p[f"{prefix}/deep/b1"]]
    deep_out, m_bwd = mlp_rows(x, ws, bs, ["silu", "identity"])
    gd = p[f"{prefix}/gate_deep"]
    gt = p[f"{prefix}/gate_dot"]
    out = x + gd * deep_out + gt * dot_out

    def bwd(g):
        grads = {}
        grads[f"{prefix}/gate_deep"] = np.array([(g * deep_out).sum()]).reshape(gd.shape)
        grads[f"{prefix}/gate_dot"] = np.array([(g * dot_out).sum()]).reshape(gt.shape)
        gdot = (g * gt).reshape(-1)
        grads[f"{prefix}/dot_map"] = np.outer(gdot, tri)
        dtri = dm.T @ gdot
        dgram = np.zeros((n_i, n_i))
        dgram[rows, cols] = dtri
        dx = g + (dgram + dgram.T) @ x
        dxm, dws, dbs = m_bwd(g * gd)
        dx = dx + dxm
        grads[f"{prefix}/deep/w0"], grads[f"{prefix}/deep/w1"] = dws
        grads[f"{prefix}/deep/b0"], grads[f"{prefix}/deep/b1"] = dbs
        return dx, grads

    return out, bwd


def global_interaction(x, summary_rows, p: dict, prefix: str, num_experts: int):
    """Experts over [X | summaries], aggregate + X residual (interaction.py:144-157)."""
    combined = np.concatenate([x] + list(summary_rows), axis=0)
    ranges = expert_ranges(combined.shape[0], num_experts)
    outs, bwds = [], []
    for i, (a, b) in enumerate(ranges):
        o, bw = wukong_expert(combined[a:b], p, f"{prefix}/expert{i}")
        outs.append(o)
        bwds.append(bw)
    stacked = np.concatenate(outs, axis=0)
    agg = p[f"{prefix}/aggregate"]
    y = agg @ stacked + x

    def bwd(g):
        grads = {f"{prefix}/aggregate": g @ stacked.T}
        dstk = agg.T @ g
        dcomb = np.zeros_like(combined)
        for (a, b), bw in zip(ranges, bwds):
            dxi, gr = bw(dstk[a:b])
            dcomb[a:b] += dxi
            grads.update(gr)
        dx = g + dcomb[: x.shape[0]]
        drows = []
        off = x.shape[0]
        for r in summary_rows:
            drows.append(dcomb[off: off + r.shape[0]])
            off += r.shape[0]
        return dx, drows, grads

    return y, bwd


def merge_grads(dst: dict, src: dict) -> None:
    for k, v in src.items():
        _acc(dst, k, v)


def zero_like_grads(p: dict) -> dict:
    return defaultdict(float)


# ---------------------------------------------------------------------------
# Ablation baselines (Table 2)
# ---------------------------------------------------------------------------


def pffn_original(x_sum, s, p: dict, prefix: str, hidden_act: str = "silu"):
    """Original PFFN: a per-sample (d, d) transform f = reshape(W2 act(W1
    flat(X_sum) + b1) + b2, (d, d)) applied rowwise, Y = S f^T, no residual
    (gdpa.py:227-257).  Returns (Y, bwd) with bwd(g) -> (dS, dX_sum, grads)."""
    from .ops import act_dfn, act_fwd

    w1, b1 = p[f"{prefix}/w1"], p[f"{prefix}/b1"]
    w2, b2 = p[f"{prefix}/w2"], p[f"{prefix}/b2"]
    d = s.shape[1]
    flat = x_sum.reshape(-1)
    pre = w1 @ flat + b1
    h = act_fwd(hidden_act, pre)
    f = (w2 @ h + b2).reshape(d, d)
    y = s @ f.T

    def bwd(g):
        df = g.T @ s                      # (d, d): dY = S f^T -> df = g^T S
        ds = g @ f
        dfv = df.reshape(-1)
        grads = {f"{prefix}/w2": np.outer(dfv, h), f"{prefix}/b2": dfv.copy()}
        dh = w2.T @ dfv
        dpre = dh * act_dfn(hidden_act, pre, h)
        grads[f"{prefix}/w1"] = np.outer(dpre, flat)
        grads[f"{prefix}/b1"] = dpre
        dflat = w1.T @ dpre
        return ds, dflat.reshape(x_sum.shape), grads

    return y, bwd


def pma_summarize(s, p: dict, prefix: str, budget: int):
    """The "w/o HSP (use PMA)" summary of PAPER.md Table 2: [CLS | PMA tokens |
    recent], the middle n_tok rows pooled by learnable queries
    (pma = MHA(Q_learn, S, S), seqsum.py:26-34) instead of
    seed attention + SumKronLinear.  Empty sequences give zeros."""
    n_cls, n_tok, n_rec = split_for_budget(budget)
    d = s.shape[1]
    parts, bwds = [], []
    for key, n in (("cls", n_cls), ("pma", n_tok)):
        if n == 0:
            continue
        if s.shape[0] == 0:
            parts.append(np.zeros((n, d)))
            bwds.append(None)
            continue
        q = p[f"{prefix}/{key}_queries"]
        o, ob = multi_head_attention(q, s, p, f"{prefix}/{key}_attn")
        parts.append(o)
        bwds.append((key, n, ob))
    rec, r_bwd = recent_rows(s, n_rec)
    parts.append(rec)
    rows = np.concatenate(parts, axis=0)

    def bwd(g):
        grads = {}
        ds = np.zeros_like(s)
        off = 0
        for entry, part in zip(bwds, parts[:len(bwds)]):
            n = part.shape[0]
            if entry is not None:
                key, _, ob = entry
                dq, dkv, gr = ob(g[off:off + n])
                merge_grads(grads, gr)
                _acc(grads, f"{prefix}/{key}_queries", dq)
                ds = ds + dkv
            off += n
        ds = ds + r_bwd(g[off:])
        return ds, grads

    return rows, bwd
