"""Kernel parity on the B200: every device op and the composed model vs the
float64 numpy oracle (itself pinned to the reference's golden vectors).

Metric: relative error = max|gpu - oracle| / max|oracle| per tensor.
Tolerances (BASELINE.json north_star): FP32 path <= 1e-5, BF16 path <= 2e-2.
"""

import ctypes as C

import numpy as np
import pytest
import torch

from oracle import kunlun as K
from oracle import model as OM

pytestmark = pytest.mark.gpu

TOL = {torch.float32: 1e-5, torch.bfloat16: 2e-2}
DTYPES = [torch.float32, torch.bfloat16]


def rel(a, b):
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if b.size == 0:
        return 0.0
    den = np.abs(b).max()
    if den == 0:
        return float(np.abs(a).max())
    return float(np.abs(a - b).max() / den)


def relf(a, b):
    """Frobenius-relative error (the norm-wise rule of oracle/parity.py)."""
    a = a.detach().double().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / den) if den > 0 else float(np.linalg.norm(a))


def check_grads(got, ref, dtype):
    """Parameter-gradient parity with the rule of oracle/parity.py."""
    from oracle.parity import grad_errors

    vals = {k: got(k).detach().double().cpu().numpy() for k in ref}
    errs = grad_errors(vals, ref, dtype == torch.float32)
    bad = sorted(((e, k) for k, e in errs.items() if not e < TOL[dtype]), reverse=True)
    assert not bad, [(k, f"{e:.3e}") for e, k in bad[:12]]
    return max(errs.values()) if errs else 0.0


def _round(x, dtype):
    return torch.tensor(np.asarray(x)).to(dtype).double().numpy()


def dev(x, dtype=torch.float32, grad=False):
    t = torch.tensor(np.asarray(x), dtype=dtype, device="cuda")
    return t.requires_grad_(grad)


@pytest.fixture(autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_10016_b200 import _capi

    _capi.lib()


# ---------------------------------------------------------------------------
# generic GEMM vs a torch fp32 reference of the same op


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("M,N,K", [(1, 1, 1), (7, 5, 3), (64, 64, 64), (130, 200, 70), (256, 384, 256),
                                   (1000, 96, 40)])
def test_gemm_plain(dtype, M, N, K):
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(M * 7 + N)
    A = torch.randn(M, K, device="cuda", generator=g).to(dtype)
    B = torch.randn(K, N, device="cuda", generator=g).to(dtype)
    ref = A.double() @ B.double()
    out = gemm(A, B, out_dtype=torch.float32)
    assert rel(out, ref.cpu().numpy()) < (1e-6 if dtype == torch.float32 else 1e-2)
    # transposed operand layouts
    out2 = gemm(A.t().contiguous().t(), B.t().contiguous().t(), out_dtype=torch.float32)
    assert rel(out2, ref.cpu().numpy()) < (1e-6 if dtype == torch.float32 else 1e-2)


@pytest.mark.parametrize("dtype", DTYPES)
def test_gemm_batched_reduce_epilogue(dtype):
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(3)
    A = torch.randn(3, 4, 33, 20, device="cuda", generator=g).to(dtype)
    B = torch.randn(1, 4, 20, 48, device="cuda", generator=g).to(dtype)
    ref = (A.double() @ B.double()).sum(0, keepdim=True)
    out = gemm(A, B, out_dtype=torch.float32, reduce=(True, False))
    tol = 1e-6 if dtype == torch.float32 else 1e-2
    assert out.shape == (1, 4, 33, 48)
    assert rel(out, ref.cpu().numpy()) < tol
    # epilogue: act(alpha*acc + bias) + beta*C + R with per-column-group codes and row limit
    Cin = torch.randn(3, 4, 33, 48, device="cuda", generator=g)
    R = torch.randn(3, 4, 33, 48, device="cuda", generator=g)
    bias = torch.randn(48, device="cuda", generator=g)
    lim = torch.tensor([33, 10, 0], device="cuda", dtype=torch.int32)
    out = Cin.clone()
    pre = torch.empty_like(out)
    gemm(A, B, out, alpha=0.5, beta=1.0, bias=bias, acts=["silu", "tanh", "relu"], act_group=16, aux=pre, aux_mode=1,
         residual=R, row_limit=lim.repeat_interleave(4))
    z = 0.5 * (A.double() @ B.double()) + bias.double()
    act = torch.cat([torch.nn.functional.silu(z[..., :16]), torch.tanh(z[..., 16:32]), torch.relu(z[..., 32:])], -1)
    full = act + Cin.double() + R.double()
    rows = torch.arange(33, device="cuda")[None, None, :, None]
    full = torch.where(rows < lim.view(3, 1, 1, 1), full, torch.zeros_like(full))
    assert rel(out, full.cpu().numpy()) < tol
    assert rel(pre, torch.where(rows < lim.view(3, 1, 1, 1), z, torch.zeros_like(z)).cpu().numpy()) < tol


# ---------------------------------------------------------------------------


def _params_gdpa(dtype, H=4, d=32, n_kv=4, n_sum=2, n_ctx=5, T=20, seed=0, acts=()):
    from paper_2602_10016_b200 import gdpa as G
    from paper_2602_10016_b200.tensor import Params

    rng = np.random.default_rng(seed)
    P = Params()
    cfg = G.GdpaConfig(dim=d, heads=H, n_kv=n_kv, tau=float(T), activations=tuple(acts))
    wg = G.WeightGenParams.create(P, "g", cfg, n_sum, d, rng)
    P.add("pool", rng.normal(0, 1 / np.sqrt(n_ctx), (n_sum, n_ctx)))
    P.finalize("cuda", dtype)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    return P, cfg, wg, named


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("H,d,n_kv,T,acts", [(4, 32, 4, 20, ()),
                                             (4, 128, 16, 300, ("silu", "relu", "identity", "tanh")),
                                             (4, 256, 16, 1024, ("silu", "relu", "identity", "tanh")),
                                             (4, 256, 16, 257, ("tanh", "silu", "sigmoid", "identity")),
                                             (2, 256, 32, 128, ("silu", "relu")),
                                             (8, 512, 16, 700, ("silu", "relu", "identity", "tanh") * 2)])
def test_gdpa_vs_oracle(dtype, H, d, n_kv, T, acts):
    """GDPA (weight generation + folded core) vs the oracle, per tensor.

    In bf16, d in {128, 256} with H*n_kv = 64 and the default activation
    cycle (incl. relu) runs the fused tcgen05 kernels — asserted through the
    kernel-path counters — including a multi-tile T = 1024 walk; the sigmoid
    case runs the GEMM composition (the fused kernels take the default cycle
    only) and asserts that instead.  bf16 tensors are compared in the
    Frobenius norm (oracle/parity.py)."""
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200 import gdpa as G

    n_sum, n_ctx = 2, 5
    P, cfg, wg, named = _params_gdpa(dtype, H, d, n_kv, n_sum, n_ctx, T, acts=acts)
    rng = np.random.default_rng(1)
    lengths = np.array([T, 7, 0, 1, max(T - 130, 1)])
    B = len(lengths)
    S = rng.normal(0, 1 / np.sqrt(d), (B, T, d))
    X = rng.normal(0, 1, (B, n_ctx, d))
    R = rng.normal(0, 1, (B, T, d))
    if dtype == torch.bfloat16:
        # identical inputs: the oracle sees the bf16 values the device reads
        # (weights: the fp32 masters, as everywhere)
        S, X, R = _round(S, dtype), _round(X, dtype), _round(R, dtype)
    S_t, X_t = dev(S, grad=True), dev(X, grad=True)
    from paper_2602_10016_b200 import _capi

    _capi.reset_path_hits()
    xs = G.summarize_nonseq(F.cast(X_t, dtype), F.PRef(P, "pool"))
    y = G.gdpa_forward(F.cast(S_t, dtype), xs, cfg, wg, lengths=lengths)
    P.zero_grad()
    (F.cast(y, torch.float32) * dev(R)).sum().backward()
    hits = _capi.path_hits()
    fused = (dtype == torch.bfloat16 and ((d in (128, 256) and H * n_kv == 64) or (d == 512 and H * n_kv == 128))
             and all(a in ("identity", "relu", "silu", "tanh") for a in cfg.activations))
    sfx = "512" if d == 512 else ""
    assert (hits["gdpa_fwd_tc" + sfx] > 0 and hits["gdpa_bwd_tc" + sfx] > 0) == fused, hits
    from oracle.parity import KINK_TOL, grad_errors, relu_kink, violations

    relu = dtype == torch.bfloat16 and "relu" in cfg.activations
    masks = None
    if relu:
        # the device's own relu' decisions: Z from the bf16 fold Kt the fused kernel reads
        with torch.no_grad():
            kt, _ = G.fold_kv(*G.generate_kv(xs, wg, cfg), wg)
        kt = kt.double().cpu().numpy()
    tol = TOL[dtype]
    grads, grads_m = {}, {}
    for b in range(B):
        L = lengths[b]
        xsum, xs_bwd = K.summarize_nonseq(X[b], named["pool"])
        kv, kv_bwd = K.generate_kv(xsum, named, "g", n_kv)
        yo, y_bwd = K.gdpa_forward(S[b, :L], kv, named, "g", float(T), cfg.activations)
        assert (rel if dtype == torch.float32 else relf)(y[b, :L].float(), yo) < tol
        assert rel(y[b, L:].float(), S[b, L:]) < (1e-7 if dtype == torch.float32 else 1e-2)
        ds, dkvs, gr = y_bwd(R[b, :L])
        dxs, gr2 = kv_bwd(dkvs)
        dx, dpool = xs_bwd(dxs)
        for k, v in list(gr.items()) + list(gr2.items()) + [("pool", dpool)]:
            K._acc(grads, k, v)
        err = rel if dtype == torch.float32 else relf
        assert err(S_t.grad[b, :L], ds) < tol
        assert rel(S_t.grad[b, L:], R[b, L:]) < (1e-6 if dtype == torch.float32 else 1e-2)
        if relu:
            # same oracle, relu' taken from the device's Z sign (isolates the kink)
            zdev = [S[b, :L] @ kt[b, h * n_kv:(h + 1) * n_kv].T for h in range(H)]
            _, y_bwd_m = _gdpa_masked(S[b, :L], kv, named, "g", float(T), cfg.activations, zdev)
            ds_m, dkvs_m, gr_m = y_bwd_m(R[b, :L])
            dxs_m, gr2_m = kv_bwd(dkvs_m)
            dx_m, dpool_m = xs_bwd(dxs_m)
            for k, v in list(gr_m.items()) + list(gr2_m.items()) + [("pool", dpool_m)]:
                K._acc(grads_m, k, v)
            assert relf(X_t.grad[b], dx_m) < tol
            assert relf(X_t.grad[b], dx) < KINK_TOL
        else:
            assert err(X_t.grad[b], dx) < tol
    vals = {k: P.grad(k).detach().double().cpu().numpy() for k in grads}
    kink = relu_kink(grads, lambda prefix: cfg.activations if prefix == "g" else None, pools=["pool"]) if relu else set()
    bad = violations(grad_errors(vals, grads, dtype == torch.float32), dtype == torch.float32, kink)
    assert not bad, bad[:8]
    if relu:
        bad = violations(grad_errors(vals, grads_m, False), False)
        assert not bad, ("vs the device-mask oracle", bad[:8])


def _gdpa_masked(s, kvs, p, prefix, tau, acts, zdev):
    """oracle.kunlun.gdpa_forward (gdpa.py:120-187) with the relu heads'
    derivative evaluated on ``zdev`` (Z as the device computes it, from its
    bf16 fold) instead of the exact Z: test infrastructure for the relu-kink
    exception (oracle/parity.py)."""
    from oracle.ops import act_dfn, act_fwd

    inv_tau = 1.0 / tau
    Wo = p[f"{prefix}/w_out"]
    cache, outs = [], []
    for h, (k, v) in enumerate(kvs):
        wq = p[f"{prefix}/head{h}/w_q"]
        q = s @ wq.T
        z = (q @ k.T) * inv_tau
        a = act_fwd(acts[h], z)
        outs.append(a @ v)
        cache.append((wq, q, z, a, k, v))
    cat = np.concatenate(outs, axis=1)

    def bwd(g):
        grads = {f"{prefix}/w_out": g.T @ cat}
        dcat = g @ Wo
        ds = g.copy()
        dkvs = []
        d_h = cache[0][0].shape[0]
        for h in range(len(kvs)):
            wq, q, z, a, k, v = cache[h]
            do = dcat[:, h * d_h:(h + 1) * d_h]
            dv = a.T @ do
            da = do @ v.T
            der = (zdev[h] > 0).astype(np.float64) if acts[h] == "relu" else act_dfn(acts[h], z, a)
            dz = da * der * inv_tau
            dq = dz @ k
            grads[f"{prefix}/head{h}/w_q"] = dq.T @ s
            ds = ds + dq @ wq
            dkvs.append((dz.T @ q, dv))
        return ds, dkvs, grads

    return cat @ Wo.T + s, bwd


@pytest.mark.parametrize("d,T,acts", [(256, 1024, ("silu", "relu", "identity", "tanh")),
                                      (128, 333, ("identity", "tanh", "silu", "relu")),
                                      (256, 100, ("relu", "relu", "relu", "relu"))])
def test_gdpa_fused_vs_gemm_composition(d, T, acts):
    """The fused kernels against the kl_gemm composition (Z/A through HBM) on
    the same bf16 inputs: both round A and dZ to bf16 for the second
    contraction, so they agree to bf16 output rounding."""
    from paper_2602_10016_b200 import functional as F

    torch.manual_seed(d + T)
    B, HK, n_kv = 6, 64, 16
    S = (torch.randn(B, T, d, device="cuda") / d ** 0.5).bfloat16().requires_grad_()
    Kt = (torch.randn(B, HK, d, device="cuda") / 2).bfloat16().requires_grad_()
    Vt = (torch.randn(B, HK, d, device="cuda") / 8).bfloat16().requires_grad_()
    lengths = torch.tensor([T, T - 1, 0, 1, T // 2, 129], dtype=torch.int32, device="cuda").clamp(max=T)
    G = torch.randn(B, T, d, device="cuda").bfloat16()
    outs = []
    for fused in (True, False):
        F.GDPA_FUSED = fused
        try:
            S.grad = Kt.grad = Vt.grad = None
            y = F.gdpa_core(S, Kt, Vt, lengths, acts, n_kv, 1.0 / 3.0)
            y.backward(G)
            outs.append([y.detach().float(), S.grad.float(), Kt.grad.float(), Vt.grad.float()])
        finally:
            F.GDPA_FUSED = True
    for name, a, b in zip(("Y", "dS", "dKt", "dVt"), outs[0], outs[1]):
        err = ((a - b).norm() / b.norm().clamp_min(1e-30)).item()
        assert err < 1e-2, (name, err)
    # pass-through rows are exact copies
    assert torch.equal(outs[0][0][2], S.detach()[2].float())
    assert torch.equal(outs[0][1][2], G[2].float())


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("T,w,causal,d,H", [(40, 3, False, 32, 2), (200, 64, False, 64, 4), (130, 17, True, 64, 4),
                                            (96, 200, False, 32, 2), (300, 128, False, 128, 2),
                                            (257, 100, True, 256, 4), (260, 5, False, 64, 1),
                                            (1024, 128, False, 256, 4), (384, 64, False, 128, 2),
                                            (200, 7, True, 128, 2), (700, 127, False, 128, 2)])
def test_swa_vs_oracle(dtype, T, w, causal, d, H):
    from paper_2602_10016_b200 import attention as A
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200.tensor import Params

    rng = np.random.default_rng(T + w)
    P = Params()
    mp = A.MhaParams.create(P, "m", d, H, rng)
    P.finalize("cuda", dtype)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    lengths = np.array([T, T - 1, 1, 0, max(T // 3, 1)])
    B = len(lengths)
    S = rng.normal(0, 1, (B, T, d))
    R = rng.normal(0, 1, (B, T, d))
    if dtype == torch.bfloat16:  # identical inputs: the oracle sees the bf16 values the device reads
        S = _round(S, dtype)
    S_t = dev(S, grad=True)
    y = A.mha_window(F.cast(S_t, dtype), mp, A.WindowSpec(w, causal), lengths)
    P.zero_grad()
    (F.cast(y, torch.float32) * dev(R)).sum().backward()
    tol = TOL[dtype]
    grads = {}
    for b in range(B):
        L = lengths[b]
        yo, bwd = K.mha_window(S[b, :L], named, "m", w, causal)
        assert rel(y[b, :L].float(), yo) < tol
        assert np.array_equal(y[b, L:].detach().float().cpu().numpy(),
                              F.cast(dev(S[b, L:]), dtype).float().cpu().numpy())
        ds, gr = bwd(R[b, :L])
        for k, v in gr.items():
            K._acc(grads, k, v)
        assert rel(S_t.grad[b, :L], ds) < tol
    check_grads(P.grad, grads, dtype)


def test_swa_support_bitexact():
    from paper_2602_10016_b200 import attention as A

    for T, w, causal in [(1, 0, False), (6, 2, False), (130, 64, False), (257, 128, True), (300, 5, False)]:
        lengths = np.array([T, max(T - 3, 0), 1, 0])
        sup = A.swa_support(lengths, T, w, causal)
        for b, L in enumerate(lengths):
            exp = np.zeros(T, dtype=np.int64)
            if L:
                exp[:L] = K.band_support_sizes(L, w, causal)
                assert np.array_equal(exp[:L], (K.band_mask(L, w, causal)).sum(1))
            assert np.array_equal(sup[b], exp), (T, w, causal, b)


@pytest.mark.parametrize("T,w,causal", [(1024, 128, False), (384, 128, True), (300, 64, False), (257, 5, True),
                                      (130, 0, False)])
def test_swa_tc_mask_bitexact_via_lse(T, w, causal):
    """The window / causal / length masks the tcgen05 forward kernels
    (swa_tc.cu key_band + per-row [klo, khi] clamps) actually apply,
    recovered from their log-sum-exp output and compared bit-exactly with the
    reference's band_mask / band_support_sizes / length mask
    (attention.py:96-112, 132-139).

    Pass 1: Q = K = 0, so every visible score is 0 and LSE_i = ln(#visible
    keys): round(exp(LSE)) is the per-query support size, exactly.
    Pass 2: Q e_0 = 1 and K[j, 0] = c_j, a bf16-exact pattern, so LSE_i =
    ln sum_{j visible} exp(c_j / 8) identifies WHICH keys are visible: the
    float64 prediction from the reference mask matches to 1e-5, while moving
    the band by one key changes LSE by >= 2e-3."""
    from paper_2602_10016_b200 import _capi

    H, d_h = 2, 64
    lengths = np.array([T, T - 1, 129 if T > 129 else T, 1, 0])
    B = len(lengths)
    lens = torch.tensor(lengths, dtype=torch.int32, device="cuda")
    pattern = np.array([0.0, 1.0, -1.5, 2.0, 0.5, -0.25, 1.5])
    c = pattern[np.arange(T) % len(pattern)]
    for pss in (1, 2):
        qkv = torch.zeros(B, T, 3 * H * d_h, device="cuda", dtype=torch.bfloat16)
        if pss == 2:
            qkv[:, :, 0] = 1.0                                   # Q head 0, column 0
            qkv[:, :, H * d_h] = torch.tensor(c, device="cuda")  # K head 0, column 0
        O = torch.empty(B, T, H * d_h, device="cuda", dtype=torch.bfloat16)
        LSE = torch.empty(B, H, T, device="cuda", dtype=torch.float32)
        _capi.reset_path_hits()
        _capi.call("kl_swa_fwd", C.byref(_capi.swa_args(qkv, lens, H, d_h, w, causal, O, LSE)), _capi._stream())
        assert _capi.path_hits()["swa_fwd_tc"] == 1
        lse = LSE[:, 0].double().cpu().numpy()
        for b, L in enumerate(lengths):
            mask = K.band_mask(L, w, causal) if L else np.zeros((0, 0), bool)
            if pss == 1:
                got = np.where(np.isinf(lse[b]), 0, np.rint(np.exp(np.where(np.isinf(lse[b]), 0, lse[b])))).astype(int)
                exp = np.zeros(T, dtype=int)
                exp[:L] = K.band_support_sizes(L, w, causal)
                assert np.array_equal(exp[:L], mask.sum(1))
                assert np.array_equal(got, exp), (b, np.nonzero(got != exp)[0][:5])
                assert np.all(np.isinf(lse[b, L:]))  # padding queries see no key
            else:
                pred = np.log((np.exp(c[:L] / 8.0)[None, :] * mask).sum(1)) if L else np.zeros(0)
                assert np.abs(lse[b, :L] - pred).max(initial=0.0) < 1e-5, b


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("T,d,H,n_seeds", [(37, 32, 2, 6), (1, 32, 2, 6), (300, 128, 2, 40), (257, 256, 4, 32),
                                           (130, 256, 4, 12), (256, 256, 4, 140), (384, 128, 2, 40),
                                           (300, 512, 8, 32), (1000, 512, 8, 12)])
def test_hsp_vs_oracle(dtype, T, d, H, n_seeds):
    """HSP + CLS pooling vs the oracle; d in {128, 256, 512} in bf16 runs the
    fused tcgen05 pooling kernels (kl_hsp_fwd / kl_hsp_bwd; d = 512 streams
    its operands and forms dS / dQ with GEMMs), with query tiles that straddle
    the seed / CLS boundary and a partial second tile — asserted through the
    kernel-path counters.  T % 8 == 0 (256, 384) takes the d <= 256
    backward's TMA-stored dZ / dS rows; the other lengths its row stores."""
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200 import seqsum as Q
    from paper_2602_10016_b200.tensor import Params

    budget, rank = 8, 2
    rng = np.random.default_rng(5)
    P = Params()
    sp = Q.SummarizerParams.create(P, "s", d, Q.SummarySplit.for_budget(budget), n_seeds, rank, H, rng)
    P.finalize("cuda", dtype)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    lengths = np.array([T, 0, max(T - 5, 1), 1])
    B = len(lengths)
    S = rng.normal(0, 1, (B, T, d)) * (4.0 / np.sqrt(d) if d > 32 else 1.0)
    R = rng.normal(0, 1, (B, budget, d))
    if dtype == torch.bfloat16:
        S = _round(S, dtype)
    S_t = dev(S, grad=True)
    from paper_2602_10016_b200 import _capi

    _capi.reset_path_hits()
    rows = Q.hsp_summarize(F.cast(S_t, dtype), sp, lengths).rows()
    P.zero_grad()
    (F.cast(rows, torch.float32) * dev(R)).sum().backward()
    hits = _capi.path_hits()
    fused = dtype == torch.bfloat16 and d in (128, 256, 512)
    assert (hits["hsp_fwd_tc"] > 0 and hits["hsp_bwd_tc"] > 0 and hits["colsoftmax"] == 0) == fused, hits
    tol = TOL[dtype]
    grads = {}
    for b in range(B):
        L = lengths[b]
        ro, bwd = K.hsp_summarize(S[b, :L], named, "s", budget)
        assert rel(rows[b].float(), ro) < tol
        ds, gr = bwd(R[b])
        for k, v in gr.items():
            K._acc(grads, k, v)
        assert rel(S_t.grad[b, :L], ds) < tol
        assert float(S_t.grad[b, L:].abs().max() if L < T else 0.0) == 0.0
    check_grads(P.grad, grads, dtype)


@pytest.mark.parametrize("dtype", DTYPES)
def test_gi_vs_oracle(dtype):
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200 import interaction as I
    from paper_2602_10016_b200.tensor import Params

    d, n_ctx, experts, hidden = 16, 5, 2, 32
    budgets = [8, 4]
    total = n_ctx + sum(budgets)
    rng = np.random.default_rng(9)
    P = Params()
    ip = I.InteractionParams.create(P, "gi", I.ExpertPartition.contiguous(total, experts), n_ctx, d, hidden, rng)
    P.finalize("cuda", dtype)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    B = 3
    X = rng.normal(0, 1, (B, n_ctx, d))
    Rows = [rng.normal(0, 1, (B, b, d)) for b in budgets]
    if dtype == torch.bfloat16:
        X, Rows = _round(X, dtype), [_round(r, dtype) for r in Rows]
    Rc = rng.normal(0, 1, (B, n_ctx, d))
    X_t = dev(X, grad=True)
    rows_t = [dev(r, grad=True) for r in Rows]
    y = I.global_interaction(F.cast(X_t, dtype), [F.cast(r, dtype) for r in rows_t], ip)
    P.zero_grad()
    (F.cast(y, torch.float32) * dev(Rc)).sum().backward()
    tol = TOL[dtype]
    grads = {}
    for b in range(B):
        yo, bwd = K.global_interaction(X[b], [r[b] for r in Rows], named, "gi", experts)
        assert rel(y[b].float(), yo) < tol
        dx, drows, gr = bwd(Rc[b])
        for k, v in gr.items():
            K._acc(grads, k, v)
        assert rel(X_t.grad[b], dx) < tol
        for e in range(2):
            assert rel(rows_t[e].grad[b], drows[e]) < tol
    check_grads(P.grad, grads, dtype)


# ---------------------------------------------------------------------------


def _spec(compskip, d=16, heads=4):
    return OM.ModelSpec(L=2, d=d, heads=heads, n_ctx=5, n_sum=2, n_kv=4, experts=2, compskip=compskip,
                        events=[OM.EventSpec(T=12, w=3, budget=8, n_seeds=6, rank=2),
                                OM.EventSpec(T=9, w=2, budget=4, n_seeds=3, rank=1)])


def _gpu_model(spec, dtype):
    from paper_2602_10016_b200.model import EventConfig, KunlunModel, ModelConfig

    cfg = ModelConfig(L=spec.L, d=spec.d, heads=spec.heads, n_ctx=spec.n_ctx, n_sum=spec.n_sum, n_kv=spec.n_kv,
                      experts=spec.experts, compskip=spec.compskip,
                      events=[EventConfig(T=e.T, w=e.w, budget=e.budget, n_seeds=e.n_seeds, rank=e.rank)
                              for e in spec.events])
    return KunlunModel(cfg, "cuda", dtype)


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("compskip", [False, True])
def test_model_vs_oracle(dtype, compskip):
    """full 2-layer, 2-event model with a parity loss that
    touches every layer output (so dead branches' backward kernels run too)."""
    from paper_2602_10016_b200 import functional as F

    spec = _spec(compskip)
    pnp = OM.init_params(spec, seed=11)
    model = _gpu_model(spec, dtype)
    model.P.load(pnp)
    rng = np.random.default_rng(4)
    B = 3
    lengths = [np.array([12, 5, 0]), np.array([9, 1, 9])]
    X = rng.normal(0, 1 / np.sqrt(spec.d), (B, spec.n_ctx, spec.d))
    S = [rng.normal(0, 1 / np.sqrt(spec.d), (B, ev.T, spec.d)) for ev in spec.events]
    if dtype == torch.bfloat16:  # identical inputs: the oracle sees the bf16 values the device reads
        X, S = _round(X, dtype), [_round(s, dtype) for s in S]
    labels = (rng.random(B) < 0.4).astype(np.float64)
    cot = [{"X": rng.normal(0, 0.1, X.shape), "S": [rng.normal(0, 0.1, s.shape) for s in S],
            "H": [rng.normal(0, 0.1, (B, ev.budget, spec.d)) for ev in spec.events]} for _ in range(spec.L)]
    ref = OM.model_forward_backward(spec, pnp, X, S, lengths, labels, cot)

    X_t = dev(X, grad=True)
    S_t = [dev(s, grad=True) for s in S]
    lens = [torch.tensor(L, dtype=torch.int32, device="cuda") for L in lengths]
    logits, outs = model.forward(F.cast(X_t, dtype), [F.cast(s, dtype) for s in S_t], lens, keep_outputs=True,
                                 prune_dead=False)
    loss = F.bce_with_logits(logits, dev(labels))
    for l, (xo, so, ho) in enumerate(outs):
        loss = loss + (F.cast(xo, torch.float32) * dev(cot[l]["X"])).sum()
        for e in range(2):
            loss = loss + (F.cast(so[e], torch.float32) * dev(cot[l]["S"][e])).sum()
            loss = loss + (F.cast(ho[e], torch.float32) * dev(cot[l]["H"][e])).sum()
    model.P.zero_grad()
    loss.backward()
    tol = TOL[dtype]
    assert rel(logits, ref["logits"]) < tol
    assert abs(float(loss) - ref["loss"]) / max(1.0, abs(ref["loss"])) < tol
    assert rel(X_t.grad, ref["dX"]) < tol
    for e in range(2):
        assert rel(S_t[e].grad, ref["dS"][e]) < tol
    check_grads(model.P.grad, ref["grads"], dtype)


@pytest.mark.parametrize("n", [2, 4, 257, 4096, 100_000])
@pytest.mark.parametrize("from_logits", [False, True])
def test_normalized_entropy(n, from_logits):
    """kl_ne vs the oracle, fp64 accumulation."""
    from oracle import ops
    from paper_2602_10016_b200.metrics import normalized_entropy

    rng = np.random.default_rng(n)
    z = (rng.normal(size=n) * 3).astype(np.float32)
    y = (rng.random(n) < 0.3).astype(np.float32)
    y[0], y[1] = 1.0, 0.0  # non-degenerate
    p = z if from_logits else (1 / (1 + np.exp(-z.astype(np.float64)))).astype(np.float32)
    got = normalized_entropy(torch.tensor(y, device="cuda"), torch.tensor(p, device="cuda"), from_logits=from_logits)
    ref = ops.normalized_entropy(y, p, from_logits=from_logits)
    for k in ("cross_entropy", "background_entropy", "ne", "ctr"):
        assert abs(getattr(got, k) - ref[k]) <= 1e-10 * max(1.0, abs(ref[k])), k
    assert got.n == n


def test_normalized_entropy_spec_examples_and_errors():
    from paper_2602_10016_b200.metrics import normalized_entropy

    def ne(y, p):
        return normalized_entropy(torch.tensor(y, device="cuda", dtype=torch.float32),
                                  torch.tensor(p, device="cuda", dtype=torch.float32)).ne

    assert abs(ne([1, 0, 1, 0], [0.5] * 4) - 1.0) < 1e-12
    assert ne([1, 0], [1 - 1e-12, 1e-12]) < 1e-10
    assert abs(ne([1, 0, 0, 0], [0.7, 0.1, 0.1, 0.1]) - 0.2991) < 5e-5
    with pytest.raises(ValueError, match="degenerate background entropy"):
        ne([0, 0, 0], [0.2, 0.3, 0.4])


@pytest.mark.parametrize("tag", ["prev", "latest", "nots", "custom", "empty"])
def test_rote_golden(tag):
    """kl_rote (fp32) vs the reference's own rote_sequence outputs / input gradients (tests/golden/rote.npz)."""
    import os

    from paper_2602_10016_b200.preproc import RoteConfig, rote_sequence

    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "rote.npz"))
    cfg = RoteConfig(z[f"{tag}:pos"], z[f"{tag}:temp"], float(z[f"{tag}:tau_scale"]),
                     "previous" if int(z[f"{tag}:mode"]) == 0 else "latest")
    s = torch.tensor(z[f"{tag}:S"], device="cuda", dtype=torch.float32, requires_grad=True)
    ts = z[f"{tag}:ts"] if int(z[f"{tag}:has_ts"]) else None
    y = rote_sequence(s, ts, cfg)
    assert tuple(y.shape) == z[f"{tag}:Y"].shape
    if y.numel():
        y.backward(torch.tensor(z[f"{tag}:cot"], device="cuda", dtype=torch.float32))
        assert rel(y, z[f"{tag}:Y"]) <= TOL[torch.float32]
        assert rel(s.grad, z[f"{tag}:dS"]) <= TOL[torch.float32]


@pytest.mark.parametrize("dtype", DTYPES)
@pytest.mark.parametrize("mode", ["previous", "latest"])
@pytest.mark.parametrize("B,T,d", [(5, 33, 16), (2, 4096, 512), (3, 37, 24), (4, 29, 12)])
def test_rote_batched(dtype, mode, B, T, d):
    """Padded batch with per-sample lengths and timestamps vs the oracle per sample; padded rows pass through."""
    from oracle import ops
    from paper_2602_10016_b200.preproc import RoteConfig, rote_sequence

    rng = np.random.default_rng(B * T + d)
    cfg = RoteConfig.default(d, tau_scale=45.0, gap_mode=mode)
    x = rng.normal(size=(B, T, d))
    ts = np.cumsum(rng.exponential(300.0, (B, T)), axis=1)
    lens = np.array([T, 0, 1] + list(rng.integers(1, T + 1, B)))[:B].astype(np.int32)
    xt = torch.tensor(x, device="cuda", dtype=dtype, requires_grad=True)
    xq = xt.detach().double().cpu().numpy()  # the inputs the kernel sees (bf16-rounded)
    y = rote_sequence(xt, ts, cfg, lengths=torch.tensor(lens, device="cuda"))
    g = rng.normal(size=(B, T, d))
    y.backward(torch.tensor(g, device="cuda", dtype=dtype))
    gq = torch.tensor(g, dtype=dtype).double().numpy()
    for b in range(B):
        n = int(lens[b])
        yo, bwd = ops.rote_sequence(xq[b, :n], ts[b, :n], cfg.pos_freqs, cfg.temp_freqs, cfg.tau_scale, mode)
        if n:
            assert rel(y[b, :n], yo) <= TOL[dtype]
            assert rel(xt.grad[b, :n], bwd(gq[b, :n])) <= TOL[dtype]
        assert torch.equal(y[b, n:], xt.detach()[b, n:])


def test_rote_errors():
    from paper_2602_10016_b200.preproc import RoteConfig, rote_sequence
    from paper_2602_10016_b200.tensor import ShapeError

    with pytest.raises(ShapeError):
        rote_sequence(torch.zeros(4, 6, device="cuda"), None, RoteConfig.default(8))
    with pytest.raises(ValueError):
        RoteConfig.default(7)
    with pytest.raises(ValueError):
        RoteConfig(np.ones(2), np.ones(3))


@pytest.mark.parametrize("grid", [None, "3"])
def test_gdpa512_fused_vs_gemm_composition(grid, monkeypatch):
    """d = 512 fused kernels (streamed operands, two 256-column halves) vs the
    kl_gemm composition, including CTAs that walk several tiles (grid
    capped through KL_GDPA_GRID) and jagged lengths."""
    from paper_2602_10016_b200 import _capi
    from paper_2602_10016_b200 import functional as F

    if grid:
        monkeypatch.setenv("KL_GDPA_GRID", grid)
    torch.manual_seed(5)
    B, T, d, HK, n_kv = 5, 1000, 512, 128, 16
    acts = ("silu", "relu", "identity", "tanh") * 2
    S = (torch.randn(B, T, d, device="cuda") / d ** 0.5).bfloat16().requires_grad_()
    Kt = (torch.randn(B, HK, d, device="cuda") / 2).bfloat16().requires_grad_()
    Vt = (torch.randn(B, HK, d, device="cuda") / 8).bfloat16().requires_grad_()
    lengths = torch.tensor([T, T - 1, 0, 1, 129], dtype=torch.int32, device="cuda")
    G = torch.randn(B, T, d, device="cuda").bfloat16()
    outs = []
    for fused in (True, False):
        F.GDPA_FUSED = fused
        try:
            S.grad = Kt.grad = Vt.grad = None
            _capi.reset_path_hits()
            y = F.gdpa_core(S, Kt, Vt, lengths, acts, n_kv, 1.0 / 3.0)
            y.backward(G)
            torch.cuda.synchronize()
            hits = _capi.path_hits()
            assert (hits["gdpa_fwd_tc512"] > 0 and hits["gdpa_bwd_tc512"] > 0) == fused, hits
            outs.append([y.detach().float(), S.grad.float(), Kt.grad.float(), Vt.grad.float()])
        finally:
            F.GDPA_FUSED = True
    for name, a, b in zip(("Y", "dS", "dKt", "dVt"), outs[0], outs[1]):
        err = ((a - b).norm() / b.norm().clamp_min(1e-30)).item()
        assert err < 1e-2, (name, err)
    assert torch.equal(outs[0][0][2], S.detach()[2].float())  # length-0 sample passes through
    assert torch.equal(outs[0][1][2], G[2].float())


@pytest.mark.parametrize("env", [None, ("KL_HSP_GRID", "5"), ("KL_HSP_CPL", "1"), ("KL_HSP_CPL", "3"),
                                 ("KL_HSP_CPL", "7")])
def test_hsp512_fused_vs_composition(env, monkeypatch):
    """d = 512 fused pooling vs the GEMM + column-softmax composition, with
    jagged lengths: the balanced forward (key blocks of each (query tile,
    half) lane split over 1 / 3 / 7 / the default number of CTAs — samples cut
    between CTAs merge their partials) and the one-CTA-per-item forward with
    CTAs walking several items (KL_HSP_GRID)."""
    from paper_2602_10016_b200 import _capi
    from paper_2602_10016_b200 import functional as F

    if env:
        monkeypatch.setenv(*env)
    balanced = not (env and env[0] == "KL_HSP_GRID")
    monkeypatch.setattr(F, "HSP_BALANCED", balanced)
    _capi.reset_path_hits()
    torch.manual_seed(6)
    B, T, d, HQ = 5, 900, 512, 320
    S = (torch.randn(B, T, d, device="cuda") * 4 / d ** 0.5).bfloat16().requires_grad_()
    Q = (torch.randn(HQ, d, device="cuda") / d ** 0.5).requires_grad_()
    lengths = torch.tensor([T, 0, 257, 1, T - 3], dtype=torch.int32, device="cuda")
    outs = []
    for fused in (True, False):
        F.HSP_FUSED = fused
        try:
            S.grad = Q.grad = None
            o1, o2 = F.hsp_pool(S, Q, lengths, splits=(256, 64))
            g1 = torch.randn_like(o1.float(), generator=torch.Generator(device="cuda").manual_seed(1)).bfloat16()
            g2 = torch.randn_like(o2.float(), generator=torch.Generator(device="cuda").manual_seed(2)).bfloat16()
            torch.autograd.backward([o1, o2], [g1, g2])
            outs.append([o1.detach().float(), o2.detach().float(), S.grad.float(), Q.grad.float()])
            if fused:
                assert (_capi.path_hits()["hsp_fwd_split"] > 0) == balanced
        finally:
            F.HSP_FUSED = True
    for name, a, b in zip(("O1", "O2", "dS", "dQ"), outs[0], outs[1]):
        err = ((a - b).norm() / b.norm().clamp_min(1e-30)).item()
        assert err < 1e-2, (name, err)


def _gdpa_setup(acts, scale=1.0, d=128, T=200):
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200 import gdpa as G

    P, cfg, wg, named = _params_gdpa(torch.bfloat16, 4, d, 16, 2, 5, T, acts=acts)
    rng = np.random.default_rng(3)
    S = torch.tensor(rng.normal(0, scale, (2, T, d)), device="cuda").bfloat16()
    X = torch.tensor(rng.normal(0, 1, (2, 5, d)), device="cuda").bfloat16()
    xs = G.summarize_nonseq(X, F.PRef(P, "pool"))
    return G, cfg, wg, S, xs


@pytest.mark.parametrize("tag", ["exp", "log", "sqrt"])
def test_numerics_error_eager(tag):
    """exp / log / sqrt GDPA heads on ordinary score ranges give Inf / NaN:
    in eager mode the op raises NumericsError (tensor.py:21-27), as the
    reference's _ensure_finite does."""
    from paper_2602_10016_b200.tensor import NumericsError, numerics_check_mode, set_numerics_check

    G, cfg, wg, S, xs = _gdpa_setup((tag, "silu", "relu", tag), scale=40.0 if tag == "exp" else 1.0)
    cfg.tau = 1e-3 if tag == "exp" else cfg.tau  # large scores: exp overflows
    old = numerics_check_mode()
    set_numerics_check("eager")
    try:
        with pytest.raises(NumericsError):
            G.gdpa_forward(S, xs, cfg, wg)
        # finite inputs with smooth heads pass
        cfg2 = G.GdpaConfig(cfg.dim, cfg.heads, cfg.n_kv, 200.0, ("silu", "relu", "identity", "tanh"))
        G.gdpa_forward(S / 40.0 if tag == "exp" else S, xs, cfg2, wg)
    finally:
        set_numerics_check(old)


def test_numerics_error_deferred_training_step():
    """Deferred mode: a NaN input leaves the training step running (no sync)
    and raise_if_nonfinite / TrainStep.check_numerics raise afterwards."""
    from paper_2602_10016_b200.configs import c1
    from paper_2602_10016_b200.model import KunlunModel
    from paper_2602_10016_b200.optim import FlatAdam, TrainStep
    from paper_2602_10016_b200.synth import ctr_batch
    from paper_2602_10016_b200.tensor import NumericsError

    cfg, _ = c1()
    B = 4
    model = KunlunModel(cfg, "cuda", torch.bfloat16, seed=0)
    Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=3)
    X = torch.tensor(Xn, device="cuda").bfloat16()
    S = [torch.tensor(s, device="cuda").bfloat16() for s in Sn]
    lens = [torch.tensor(l, device="cuda") for l in Ln]
    y = torch.tensor(yn, device="cuda")
    step = TrainStep(model, FlatAdam(model.P), X, S, lens, y, None)
    step.eager()
    step.check_numerics()  # clean
    S[0][1, 3, 5] = float("nan")
    step.eager()
    with pytest.raises(NumericsError):
        step.check_numerics()
    step.check_numerics()  # the flag was cleared


@pytest.mark.parametrize("dtype", DTYPES)
def test_gdpa_forward_jagged_vs_oracle(dtype):
    """gdpa_forward_jagged (gdpa.py:209-224): one batched launch over the
    padded layout of a JaggedBatch (lengths 0, 1, T and between), per-sample
    context summaries; forward only, zero-length samples pass through."""
    from paper_2602_10016_b200 import gdpa as G
    from paper_2602_10016_b200.jagged import JaggedBatch

    d, H, n_kv, n_sum = 32, 4, 4, 2
    P, cfg, wg, named = _params_gdpa(dtype, H, d, n_kv, n_sum, 5, 40)
    rng = np.random.default_rng(4)
    lens = [40, 0, 1, 17, 40]
    vals = [rng.normal(0, 1 / np.sqrt(d), (n, d)) for n in lens]
    if dtype == torch.bfloat16:
        vals = [_round(v, dtype) for v in vals]
    batch = JaggedBatch(np.concatenate(vals, axis=0), np.concatenate([[0], np.cumsum(lens)]))
    xs = [_round(rng.normal(0, 1, (n_sum, d)), dtype) if dtype == torch.bfloat16 else rng.normal(0, 1, (n_sum, d))
          for _ in lens]
    out = G.gdpa_forward_jagged(batch, xs, cfg, wg)
    assert isinstance(out, JaggedBatch) and np.array_equal(out.offsets, batch.offsets)
    for b, n in enumerate(lens):
        got = out.values[out.offsets[b]:out.offsets[b + 1]]
        if n == 0:
            assert got.shape == (0, d)
            continue
        kv, _ = K.generate_kv(xs[b], named, "g", n_kv)
        yo, _ = K.gdpa_forward(vals[b], kv, named, "g", float(cfg.tau), cfg.activations)
        assert (rel if dtype == torch.float32 else relf)(got, yo) < TOL[dtype]


@pytest.mark.parametrize("dtype", DTYPES)
def test_multi_head_attention_arbitrary_mask_vs_oracle(dtype):
    """multi_head_attention with a dense boolean mask (attention.py:69-93):
    cross-attention of query rows over key rows, a random mask with one
    fully-masked query row (-> 0, tensor.py:494-498)."""
    from paper_2602_10016_b200 import attention as A
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200.tensor import Params

    d, H, n_q, n_k = 32, 4, 7, 11
    rng = np.random.default_rng(12)
    P = Params()
    mp = A.MhaParams.create(P, "m", d, H, rng)
    P.finalize("cuda", dtype)
    named = {n: P[n].double().cpu().numpy() for n in P.names()}
    xq = _round(rng.normal(0, 1, (n_q, d)), dtype) if dtype == torch.bfloat16 else rng.normal(0, 1, (n_q, d))
    xkv = _round(rng.normal(0, 1, (n_k, d)), dtype) if dtype == torch.bfloat16 else rng.normal(0, 1, (n_k, d))
    mask = rng.random((n_q, n_k)) < 0.6
    mask[3] = False
    R = rng.normal(0, 1, (n_q, d))
    q_t, kv_t = dev(xq, grad=True), dev(xkv, grad=True)
    y = A.multi_head_attention(F.cast(q_t, dtype), F.cast(kv_t, dtype), mp, mask=mask)
    P.zero_grad()
    (F.cast(y, torch.float32) * dev(R)).sum().backward()
    yo, bwd = K.multi_head_attention(xq, xkv, named, "m", mask)
    assert rel(y.float(), yo) < TOL[dtype]
    assert np.abs(y[3].detach().float().cpu().numpy()).max() == 0.0  # fully-masked row
    dxq, dxkv, gr = bwd(R)
    err = rel if dtype == torch.float32 else relf
    assert err(q_t.grad, dxq) < TOL[dtype]
    assert err(kv_t.grad, dxkv) < TOL[dtype]
    check_grads(P.grad, gr, dtype)


def test_hsp512_long_sequence_repeat():
    """The balanced d = 512 pooling forward at a bench-length sequence (T = 4096,
    32 key blocks per sample, every query tile / half lane split over many
    CTAs), three launches, against a torch fp32 evaluation: a pipeline race
    in a variant that kept P in TMEM only showed up here (and as NaN in the
    bench's training steps), not at the short parity shapes."""
    from paper_2602_10016_b200 import _capi
    from paper_2602_10016_b200 import functional as F

    torch.manual_seed(3)
    B, T, d, HQ = 6, 4096, 512, 320
    # score magnitudes growing along the sequence: the running max moves on
    # most key blocks, so the online-softmax rescale path runs constantly
    ramp = (1.0 + torch.arange(T, device="cuda") / 512.0)[None, :, None]
    S = (torch.randn(B, T, d, device="cuda") / d ** 0.5 * ramp).bfloat16()
    Q = torch.randn(HQ, d, device="cuda") * 2.0
    lengths = torch.tensor([T, T, 3000, 1, 0, T - 77], dtype=torch.int32, device="cuda")
    Z = torch.einsum("qd,btd->bqt", Q.bfloat16().float(), S.float())
    mask = torch.arange(T, device="cuda")[None, None, :] < lengths[:, None, None].long()
    P = torch.softmax(Z.masked_fill(~mask, float("-inf")), dim=-1).nan_to_num(0.0)
    ref = torch.einsum("bqt,btd->bqd", P, S.float())
    for _ in range(3):
        _capi.reset_path_hits()
        o1, o2 = F.hsp_pool(S, Q, lengths, splits=(256, 64))
        assert _capi.path_hits()["hsp_fwd_split"] > 0
        out = torch.cat([o1.float(), o2.float()], dim=1)
        assert torch.isfinite(out).all()
        assert ((out - ref).abs().max() / ref.abs().max()).item() < 2e-2
