"""tcgen05 GEMM (sm_100a) vs a torch float64 reference of the same op, over
operand majors, tails, batching, batch reduction and the fused epilogue.
The tcgen05 path is forced (kl_set_gemm_path(2)) so a shape it cannot take
fails loudly instead of silently using the SIMT kernel."""

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def force_tc():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    from paper_2602_10016_b200 import _capi

    _capi.lib().kl_set_gemm_path(2)
    yield
    _capi.lib().kl_set_gemm_path(0)


def rel(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def operand(shape, kmajor, g):
    """(…, R, C) tensor whose last dim is contiguous if kmajor else the one before."""
    t = torch.randn(*shape, device="cuda", generator=g).to(torch.bfloat16)
    if kmajor:
        return t
    return t.transpose(-1, -2).contiguous().transpose(-1, -2)


@pytest.mark.parametrize("a_k", [True, False])
@pytest.mark.parametrize("b_n", [True, False])
@pytest.mark.parametrize("M,N,K", [(128, 64, 64), (304, 160, 200), (1024, 768, 256), (64, 256, 1024), (264, 48, 72)])
def test_tc_plain(a_k, b_n, M, N, K):
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    A = operand((M, K), a_k, g)
    B = operand((K, N), b_n, g)
    ref = A.double() @ B.double()
    out = gemm(A, B, out_dtype=torch.float32)
    torch.cuda.synchronize()
    assert rel(out, ref) < 1e-5
    outb = gemm(A, B)  # bf16 output
    assert rel(outb, ref) < 1e-2


@pytest.mark.parametrize("a_k", [True, False])
def test_tc_batched_reduce(a_k):
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(7)
    A = operand((3, 4, 200, 96), a_k, g)
    B = operand((1, 4, 96, 144), True, g)
    ref = A.double() @ B.double()
    out = gemm(A, B, out_dtype=torch.float32)
    assert rel(out, ref) < 1e-5
    out = gemm(A, B, out_dtype=torch.float32, reduce=(True, False))
    assert rel(out, ref.sum(0, keepdim=True)) < 1e-5
    out = gemm(A, B.expand(3, 4, 96, 144), out_dtype=torch.float32, reduce=(True, True))
    assert rel(out, ref.sum((0, 1), keepdim=True)) < 1e-5


def test_tc_epilogue():
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(9)
    A = operand((2, 300, 128), True, g)
    B = operand((128, 96), False, g)
    R = torch.randn(2, 300, 96, device="cuda", generator=g)
    Cin = torch.randn(2, 300, 96, device="cuda", generator=g)
    bias = torch.randn(96, device="cuda", generator=g)
    lim = torch.tensor([300, 77], device="cuda", dtype=torch.int32)
    out = Cin.clone()
    pre = torch.empty_like(out)
    gemm(A, B, out, alpha=0.25, beta=1.0, bias=bias, acts=["silu", "tanh"], act_group=48, aux=pre, aux_mode=1,
         residual=R, row_limit=lim)
    z = 0.25 * (A.double() @ B.double()) + bias.double()
    act = torch.cat([torch.nn.functional.silu(z[..., :48]), torch.tanh(z[..., 48:])], -1)
    full = act + Cin.double() + R.double()
    rows = torch.arange(300, device="cuda")[None, :, None]
    keep = rows < lim.view(2, 1, 1)
    assert rel(torch.where(keep, out.double(), 0), torch.where(keep, full, 0)) < 1e-5
    assert float(out[1, 77:].abs().max()) == 0.0
    # dact mode: out = acc * act'(aux)
    d = torch.empty_like(out)
    gemm(A, B, d, acts=["silu", "tanh"], act_group=48, aux=pre, aux_mode=2)
    acc = A.double() @ B.double()
    pz = pre.double()
    s = torch.sigmoid(pz[..., :48])
    der = torch.cat([s * (1 + pz[..., :48] * (1 - s)), 1 - torch.tanh(pz[..., 48:]) ** 2], -1)
    assert rel(d, acc * der) < 1e-5


def test_tc_strided_views():
    """Operand views used by the model: head-strided W_out, transposed
    activations, permuted outputs."""
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(11)
    H, dh, d, B, n = 4, 64, 256, 8, 160
    W = torch.randn(d, d, device="cuda", generator=g).to(torch.bfloat16)
    Wv = W.view(d, H, dh).permute(1, 2, 0)  # (H, dh, d), K-major B
    V = torch.randn(B, H, n, dh, device="cuda", generator=g).to(torch.bfloat16)
    out = gemm(V, Wv, out_dtype=torch.float32)
    assert rel(out, V.double() @ Wv.double()) < 1e-5
    S = torch.randn(B, 1024, d, device="cuda", generator=g).to(torch.bfloat16)
    P = torch.randn(B, 1024, n, device="cuda", generator=g).to(torch.bfloat16)
    pooled = gemm(P.transpose(1, 2), S, out_dtype=torch.float32)  # M-major A, N-major B
    assert rel(pooled, P.double().transpose(1, 2) @ S.double()) < 1e-5
    o = torch.empty(B, n, H, dh, device="cuda", dtype=torch.float32)
    X = torch.randn(B, H, n, d, device="cuda", generator=g).to(torch.bfloat16)
    gemm(X, Wv.transpose(1, 2), o.permute(0, 2, 1, 3))
    assert rel(o.permute(0, 2, 1, 3), X.double() @ Wv.double().transpose(1, 2)) < 1e-5


@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
def test_tc_splitk_workspace(out_dtype):
    """Few output tiles + long K with a non-accumulating epilogue: split-K
    through the fp32 workspace and the reduce + epilogue pass."""
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(13)
    A = operand((128, 6144), True, g)
    B = operand((6144, 304), False, g)
    bias = torch.randn(304, device="cuda", generator=g)
    out = gemm(A, B, out_dtype=out_dtype, bias=bias, acts=["tanh"])
    ref = torch.tanh(A.double() @ B.double() + bias.double())
    assert rel(out, ref) < (1e-2 if out_dtype == torch.bfloat16 else 1e-4)  # fp32 accumulation over K=6144
    R = torch.randn(128, 304, device="cuda", generator=g).to(out_dtype)
    out = gemm(A, B, out_dtype=out_dtype, residual=R, alpha=0.5)
    ref = 0.5 * (A.double() @ B.double()) + R.double()
    assert rel(out, ref) < (1e-2 if out_dtype == torch.bfloat16 else 1e-4)  # fp32 accumulation over K=6144


@pytest.mark.gpu
@pytest.mark.parametrize("N", [96, 256, 320, 768])
def test_tc_tma_epilogue(N):
    """TMA-store epilogue (thread = row, swizzled staging boxes): bias +
    slab-uniform activations + row limit + TMA-staged residual into bf16,
    and fp32 accumulate-into-C through the TMA reduce-add (also split-K)."""
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(N)
    A = operand((3, 333, 256), True, g)
    B = operand((256, N), False, g)
    bias = torch.randn(N, device="cuda", generator=g)
    R = torch.randn(3, 333, N, device="cuda", generator=g).to(torch.bfloat16)
    lim = torch.tensor([333, 200, 0], device="cuda", dtype=torch.int32)
    z = A.double() @ B.double() * 0.5 + bias.double()
    cols = torch.arange(N, device="cuda") // 32 % 2
    act = torch.where(cols == 0, torch.nn.functional.silu(z), torch.relu(z)) + R.double()
    rows = torch.arange(333, device="cuda")[None, :, None]
    ref = torch.where(rows < lim.view(3, 1, 1), act, torch.zeros_like(act))
    out = gemm(A, B, alpha=0.5, bias=bias, acts=["silu", "relu"], act_group=32, residual=R, row_limit=lim)
    assert rel(out, ref) < 1e-2
    # fp32 C += A^T B summed over the batch (weight-gradient form)
    C0 = torch.randn(256, N, device="cuda", generator=g)
    C = C0.clone()
    gemm(A.transpose(1, 2), R, C, beta=1.0, reduce=(False, True))
    ref = C0.double() + (A.double().transpose(1, 2) @ R.double()).sum(0)
    assert rel(C, ref) < 1e-5


@pytest.mark.gpu
@pytest.mark.parametrize("N,out_dtype", [(256, torch.bfloat16), (320, torch.float32), (200, torch.bfloat16)])
def test_tc_tma_epilogue_aux(N, out_dtype):
    """TMA-store epilogue with the aux side output: aux_mode 1 keeps the
    pre-activation (row-limited rows zero) beside the activated C; aux_mode 2
    multiplies the product by act'(aux) (the MLP backward)."""
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(N + 7)
    A = operand((2, 333, 256), True, g)
    B = operand((256, N), False, g)
    bias = torch.randn(N, device="cuda", generator=g)
    lim = torch.tensor([333, 150], device="cuda", dtype=torch.int32)
    out = torch.empty(2, 333, N, device="cuda", dtype=out_dtype)
    pre = torch.empty(2, 333, N, device="cuda", dtype=out_dtype)
    gemm(A, B, out, bias=bias, acts=["silu"], aux=pre, aux_mode=1, row_limit=lim)
    z = A.double() @ B.double() + bias.double()
    keep = torch.arange(333, device="cuda")[None, :, None] < lim.view(2, 1, 1)
    tol = 1e-2 if out_dtype == torch.bfloat16 else 1e-5
    assert rel(pre, torch.where(keep, z, 0)) < tol
    assert rel(out, torch.where(keep, torch.nn.functional.silu(z), 0)) < (1e-2 if out_dtype == torch.bfloat16 else 2e-3)
    d = torch.empty_like(out)
    gemm(A, B, d, acts=["silu"], aux=pre, aux_mode=2)
    pz = pre.double()
    s = torch.sigmoid(pz)
    assert rel(d, (A.double() @ B.double()) * s * (1 + pz * (1 - s))) < tol


@pytest.mark.gpu
@pytest.mark.parametrize("N", [256, 320])
def test_tc_residual_long_k(N):
    """Residual epilogue with a long reduction: 256-wide tiles with a single
    TMA-staged residual buffer (issued after the tile's operand loads)."""
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(N + 11)
    A = operand((3, 333, 768), True, g)
    B = operand((768, N), False, g)
    R = torch.randn(3, 333, N, device="cuda", generator=g).to(torch.bfloat16)
    out = gemm(A, B, residual=R)
    ref = A.double() @ B.double() + R.double()
    assert rel(out, ref) < 1e-2
    C = R.clone()
    gemm(A, B, C, beta=1.0)  # accumulate onto a bf16 output: the residual path with R = C
    assert rel(C, ref) < 1e-2


@pytest.mark.parametrize("N", [96, 160, 192, 224, 384])
@pytest.mark.parametrize("out_dtype", [torch.bfloat16, torch.float32])
def test_gemm_partial_n_tiles_many_m_tiles(N, out_dtype):
    """N that splits into tiles narrower than the N range, with more M tiles
    than SMs (persistent CTAs walk several tiles): every N tile is a whole
    number of 128-byte TMA-store boxes, so no tile's store overlaps its
    neighbour's columns (regression: N = 192 at M = 8192 gave NaN / garbage
    rows from 96-column bf16 tiles, the c1 QKV projection)."""
    from paper_2602_10016_b200._capi import gemm

    torch.manual_seed(N)
    M, K = 8192, 64
    A = torch.randn(M, K, device="cuda").bfloat16()
    W = torch.randn(N, K, device="cuda").bfloat16()
    ref = A.double() @ W.double().t()
    for _ in range(3):
        c = gemm(A, W.t(), out_dtype=out_dtype)
        torch.cuda.synchronize()
        assert torch.isfinite(c).all()
        err = ((c.double() - ref).abs().max() / ref.abs().max()).item()
        assert err < 1e-2, err


@pytest.mark.parametrize("a_k,b_n", [(True, False), (False, True), (True, True)])
def test_tc_wide_pairs(a_k, b_n):
    """Wide CTA pairs (256 x 512 tiles, two N = 256 products per k step into
    one 512-column accumulator): a long-K bf16 GEMM with bias + 16-column
    activation groups + aux pre-activation + row limit, batched, M and N
    tails of the pair tile; and the fp32 accumulate weight-gradient form
    (batch-reduced, split over the SMs)."""
    from paper_2602_10016_b200 import _capi
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(11)
    M, N, K = 9000, 1024, 1600  # 2 x 18 x 2 = 72 pair tiles (>= one wave of pairs), M tail of 40 rows
    A = operand((2, M, K), a_k, g) * 0.05
    B = operand((K, N), not b_n, g) * 0.05
    bias = torch.randn(N, device="cuda", generator=g)
    lim = torch.tensor([M, 4321], device="cuda", dtype=torch.int32)
    out = torch.empty(2, M, N, device="cuda", dtype=torch.bfloat16)
    pre = torch.empty(2, M, N, device="cuda", dtype=torch.bfloat16)
    _capi.reset_path_hits()
    gemm(A, B, out, bias=bias, acts=["silu", "relu"], act_group=16, aux=pre, aux_mode=1, row_limit=lim)
    assert _capi.path_hits()["gemm_wide"] == 1
    z = A.double() @ B.double() + bias.double()
    keep = torch.arange(M, device="cuda")[None, :, None] < lim.view(2, 1, 1)
    cols = torch.arange(N, device="cuda") // 16 % 2
    act = torch.where(cols == 0, torch.nn.functional.silu(z), torch.relu(z))
    assert rel(pre, torch.where(keep, z, 0)) < 1e-2
    assert rel(out, torch.where(keep, act, 0)) < 1e-2
    # residual (C = A B + R, bf16): read by the wide epilogue from global memory
    R = torch.randn(2, M, N, device="cuda", generator=g).to(torch.bfloat16)
    _capi.reset_path_hits()
    outr = gemm(A, B, residual=R)
    assert _capi.path_hits()["gemm_wide"] == 1
    assert rel(outr, A.double() @ B.double() + R.double()) < 1e-2
    # accumulate into a bf16 C (the dX form: C += A B)
    C0 = torch.randn(2, M, N, device="cuda", generator=g).to(torch.bfloat16)
    C = C0.clone()
    gemm(A, B, C, beta=1.0)
    assert rel(C, A.double() @ B.double() + C0.double()) < 1e-2
    # weight-gradient form: C (fp32) += sum_b A_b^T D_b
    D = operand((6, 4096, 512), True, g)
    X = operand((6, 4096, 1536), a_k, g)
    C0 = torch.randn(1536, 512, device="cuda", generator=g)
    C = C0.clone()
    _capi.reset_path_hits()
    gemm(X.transpose(1, 2), D, C, beta=1.0, reduce=(False, True))
    assert _capi.path_hits()["gemm_wide"] == 1
    ref = C0.double() + (X.double().transpose(1, 2) @ D.double()).sum(0)
    assert rel(C, ref) < 1e-5


def test_gemm_fold_reduced_batch_into_k():
    """A reduced batch dim whose A columns / B rows continue across it runs as
    one long k loop (kl_gemm's batch folding; K = 40 per sample would pad each
    64-wide k block): the weight-gradient form sum_z X_z^T G_z, fp32
    accumulate and bf16 store, against fp64."""
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(21)
    X = torch.randn(6, 40, 96, device="cuda", generator=g).bfloat16()
    G = torch.randn(6, 40, 80, device="cuda", generator=g).bfloat16()
    ref = (X.double().transpose(1, 2) @ G.double()).sum(0)
    C0 = torch.randn(96, 80, device="cuda", generator=g)
    C = C0.clone()
    gemm(X.transpose(1, 2), G, C.view(1, 96, 80), beta=1.0, reduce=(False, True))
    assert rel(C, C0.double() + ref) < 1e-5
    Cb = torch.empty(1, 96, 80, device="cuda", dtype=torch.bfloat16)
    gemm(X.transpose(1, 2), G, Cb, reduce=(False, True))
    assert rel(Cb[0], ref) < 1e-2


def test_gemm_fold_broadcast_batch_into_m():
    """The opt-in M folds (KL_GEMM_FOLD=1, read once per process: run in a
    child): a per-sample M = 16 product against a broadcast weight becomes
    one 2048-row GEMM (KL_GEMM_TRACE shows the folded M) with the same
    result."""
    import os
    import subprocess
    import sys

    code = (
        "import torch, sys; sys.path.insert(0, '.');"
        "from paper_2602_10016_b200._capi import gemm;"
        "g = torch.Generator(device='cuda').manual_seed(3);"
        "A = torch.randn(128, 16, 64, device='cuda', generator=g).bfloat16();"
        "W = torch.randn(64, 256, device='cuda', generator=g).bfloat16();"
        "b = torch.randn(256, device='cuda', generator=g);"
        "C = gemm(A, W, bias=b, acts=['relu']); torch.cuda.synchronize();"
        "ref = torch.relu(A.double() @ W.double() + b.double());"
        "err = ((C.double() - ref).norm() / ref.norm()).item(); print('err', err); assert err < 1e-2")
    env = dict(os.environ, KL_GEMM_FOLD="1", KL_GEMM_TRACE="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0, r.stderr[-2000:]
    assert "gemm_tc M=2048 N=256 K=64 nb=1x1" in r.stderr, r.stderr[-2000:]


def test_tc_wide_plain_early_release():
    """Wide pairs with a plain bf16 store (MODE 2: no bias / activation /
    residual): the epilogue releases the 512-column accumulator after its
    TMEM drain, before the TMA stores (epi_wide_regs) — batched, with an M
    tail and a per-batch row limit."""
    from paper_2602_10016_b200 import _capi
    from paper_2602_10016_b200._capi import gemm

    g = torch.Generator(device="cuda").manual_seed(13)
    M, N, K = 9000, 1024, 512  # 2 x 36 x 2 = 144 pair tiles, M tail of 40 rows
    A = operand((2, M, K), True, g) * 0.05
    B = operand((K, N), False, g) * 0.05
    lim = torch.tensor([M, 3001], device="cuda", dtype=torch.int32)
    _capi.reset_path_hits()
    out = gemm(A, B, row_limit=lim)
    out2 = gemm(A, B, alpha=0.5)
    torch.cuda.synchronize()
    assert _capi.path_hits()["gemm_wide"] == 2
    z = A.double() @ B.double()
    keep = torch.arange(M, device="cuda")[None, :, None] < lim.view(2, 1, 1)
    assert rel(out, torch.where(keep, z, 0)) < 1e-2
    assert float(out[1, 3001:].abs().max()) == 0.0
    assert rel(out2, 0.5 * z) < 1e-2
