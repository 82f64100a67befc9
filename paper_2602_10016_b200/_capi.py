"""ctypes binding of libkunlun_sm100a.so (include/kunlun_capi.h).

The product path has no fallback: if the library is missing, or no CUDA
device is present when an op runs, the call raises.  Python ints/pointers
only cross the boundary — no torch types in the C signatures.
"""

from __future__ import annotations

import ctypes as C
import os

import torch

from .tensor import NumericsError, ShapeError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libkunlun_sm100a.so")
if os.environ.get("KL_LIB_PATH"):  # A/B timing of two builds in one GPU session (scripts/r2/)
    LIB_PATH = os.environ["KL_LIB_PATH"]

KL_OK, KL_EBADSHAPE, KL_EUNSUPPORTED, KL_ELAUNCH = 0, 1, 2, 3
KL_F32, KL_BF16 = 0, 1
MAX_ACT = 32

ACT_CODES = {"identity": 0, "relu": 1, "silu": 2, "tanh": 3, "sigmoid": 4, "exp": 5, "sqrt": 6, "log": 7}


class GemmArgs(C.Structure):
    _fields_ = [
        ("M", C.c_int), ("N", C.c_int), ("K", C.c_int),
        ("nb1", C.c_int), ("nb2", C.c_int), ("red1", C.c_int), ("red2", C.c_int),
        ("ab_dtype", C.c_int), ("c_dtype", C.c_int),
        ("A", C.c_void_p), ("a_rs", C.c_longlong), ("a_cs", C.c_longlong), ("a_s1", C.c_longlong), ("a_s2", C.c_longlong),
        ("B", C.c_void_p), ("b_rs", C.c_longlong), ("b_cs", C.c_longlong), ("b_s1", C.c_longlong), ("b_s2", C.c_longlong),
        ("C", C.c_void_p), ("c_rs", C.c_longlong), ("c_cs", C.c_longlong), ("c_s1", C.c_longlong), ("c_s2", C.c_longlong),
        ("R", C.c_void_p), ("r_rs", C.c_longlong), ("r_cs", C.c_longlong), ("r_s1", C.c_longlong), ("r_s2", C.c_longlong),
        ("aux", C.c_void_p), ("aux_mode", C.c_int),
        ("alpha", C.c_float), ("beta", C.c_float),
        ("bias", C.c_void_p), ("row_limit", C.c_void_p),
        ("n_act", C.c_int), ("act_group", C.c_int),
        ("act_codes", C.c_int * MAX_ACT),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_longlong),
    ]


class SwaArgs(C.Structure):
    _fields_ = [
        ("B", C.c_int), ("T", C.c_int), ("H", C.c_int), ("d_h", C.c_int),
        ("w", C.c_int), ("causal", C.c_int), ("dtype", C.c_int), ("scale", C.c_float),
        ("lengths", C.c_void_p),
        ("QKV", C.c_void_p), ("ld_qkv", C.c_longlong), ("bs_qkv", C.c_longlong),
        ("O", C.c_void_p), ("ld_o", C.c_longlong), ("bs_o", C.c_longlong),
        ("LSE", C.c_void_p),
        ("dO", C.c_void_p), ("dQKV", C.c_void_p), ("Dbuf", C.c_void_p),
    ]


class ColSoftmaxArgs(C.Structure):
    _fields_ = [
        ("Bn", C.c_int), ("T", C.c_int), ("C", C.c_int),
        ("dtype_in", C.c_int), ("dtype_out", C.c_int),
        ("X", C.c_void_p), ("x_rs", C.c_longlong), ("x_bs", C.c_longlong),
        ("P", C.c_void_p), ("p_rs", C.c_longlong), ("p_bs", C.c_longlong),
        ("LSE", C.c_void_p), ("lengths", C.c_void_p),
        ("dP", C.c_void_p), ("dp_rs", C.c_longlong), ("dp_bs", C.c_longlong),
        ("dX", C.c_void_p), ("dx_rs", C.c_longlong), ("dx_bs", C.c_longlong),
        ("dX_lo", C.c_void_p),
        ("dtype_dp", C.c_int),
        ("Dcol", C.c_void_p),
    ]


class GdpaArgs(C.Structure):
    _fields_ = [
        ("B", C.c_int), ("T", C.c_int), ("d", C.c_int), ("HK", C.c_int), ("n_kv", C.c_int),
        ("dtype", C.c_int), ("inv_tau", C.c_float), ("n_act", C.c_int),
        ("act_codes", C.c_int * MAX_ACT),
        ("lengths", C.c_void_p),
        ("S", C.c_void_p), ("s_rs", C.c_longlong), ("s_bs", C.c_longlong),
        ("Kt", C.c_void_p), ("Vt", C.c_void_p), ("Y", C.c_void_p),
        ("dY", C.c_void_p), ("dS", C.c_void_p), ("dKt", C.c_void_p), ("dVt", C.c_void_p),
        ("trace", C.c_void_p),
        ("dZ_out", C.c_void_p), ("A_out", C.c_void_p),
    ]


class RoteArgs(C.Structure):
    """kl_rote_args (include/kunlun_capi.h)."""
    _fields_ = [
        ("B", C.c_int), ("T", C.c_int), ("d", C.c_int), ("dtype", C.c_int),
        ("x", C.c_void_p), ("x_rs", C.c_longlong), ("x_bs", C.c_longlong),
        ("y", C.c_void_p), ("y_rs", C.c_longlong), ("y_bs", C.c_longlong),
        ("lengths", C.c_void_p), ("timestamps", C.c_void_p), ("ts_bs", C.c_longlong),
        ("pos_freqs", C.c_void_p), ("temp_freqs", C.c_void_p),
        ("tau_scale", C.c_double), ("gap_mode", C.c_int), ("inverse", C.c_int),
    ]


MAX_SEGS = 16


class RegroupSeg(C.Structure):
    _fields_ = [("src", C.c_void_p), ("src_bs", C.c_longlong), ("src_rs", C.c_longlong),
                ("dst", C.c_void_p), ("dst_bs", C.c_longlong), ("dst_rs", C.c_longlong), ("rows", C.c_int)]


class RegroupArgs(C.Structure):
    _fields_ = [("B", C.c_int), ("d", C.c_int), ("dtype", C.c_int), ("n_seg", C.c_int),
                ("seg", RegroupSeg * MAX_SEGS)]


class HspArgs(C.Structure):
    _fields_ = [
        ("B", C.c_int), ("T", C.c_int), ("HQ", C.c_int), ("d", C.c_int), ("n1", C.c_int),
        ("dtype", C.c_int),
        ("lengths", C.c_void_p),
        ("S", C.c_void_p), ("s_rs", C.c_longlong), ("s_bs", C.c_longlong),
        ("Q", C.c_void_p),
        ("O1", C.c_void_p), ("o1_bs", C.c_longlong),
        ("O2", C.c_void_p), ("o2_bs", C.c_longlong),
        ("LSE", C.c_void_p),
        ("dO1", C.c_void_p), ("dO2", C.c_void_p),
        ("dS", C.c_void_p), ("ds_rs", C.c_longlong), ("ds_bs", C.c_longlong),
        ("accumulate_ds", C.c_int),
        ("dZ", C.c_void_p), ("dZ_lo", C.c_void_p),
        ("Dq", C.c_void_p),
        ("q_group", C.c_int),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_longlong),
    ]


_lib = None

_SIGS = {
    "kl_version": ([], C.c_int),
    "kl_last_error": ([], C.c_char_p),
    "kl_launch_count": ([], C.c_ulonglong),
    "kl_tcgen05_available": ([], C.c_int),
    "kl_set_gemm_path": ([C.c_int], None),
    "kl_set_pdl": ([C.c_int], None),
    "kl_last_gemm_path": ([], C.c_int),
    "kl_path_hits": ([C.c_int], C.c_ulonglong),
    "kl_masked_softmax_fwd": ([C.c_longlong, C.c_int, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p],
                              C.c_int),
    "kl_masked_softmax_bwd": ([C.c_longlong, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "kl_embed_nonseq_fwd": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 5 + [C.c_longlong, C.c_void_p,
                             C.c_void_p], C.c_int),
    "kl_embed_nonseq_bwd": ([C.c_int, C.c_int, C.c_int, C.c_int, C.c_int] + [C.c_void_p] * 4 + [C.c_longlong] +
                            [C.c_void_p] * 3, C.c_int),
    "kl_reset_path_hits": ([], None),
    "kl_gemm": ([C.POINTER(GemmArgs), C.c_void_p], C.c_int),
    "kl_gdpa_fwd": ([C.POINTER(GdpaArgs), C.c_void_p], C.c_int),
    "kl_gdpa_bwd": ([C.POINTER(GdpaArgs), C.c_void_p], C.c_int),
    "kl_hsp_fwd": ([C.POINTER(HspArgs), C.c_void_p], C.c_int),
    "kl_hsp_fwd_workspace_bytes": ([C.POINTER(HspArgs)], C.c_longlong),
    "kl_hsp_bwd": ([C.POINTER(HspArgs), C.c_void_p], C.c_int),
    "kl_swa_fwd": ([C.POINTER(SwaArgs), C.c_void_p], C.c_int),
    "kl_swa_bwd": ([C.POINTER(SwaArgs), C.c_void_p], C.c_int),
    "kl_swa_debug_support": ([C.POINTER(SwaArgs), C.c_void_p, C.c_void_p], C.c_int),
    "kl_colsoftmax_fwd": ([C.POINTER(ColSoftmaxArgs), C.c_void_p], C.c_int),
    "kl_colsoftmax_bwd": ([C.POINTER(ColSoftmaxArgs), C.c_void_p], C.c_int),
    "kl_rmsnorm_fwd": ([C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
    "kl_rmsnorm_bwd": ([C.c_int, C.c_int, C.c_float] + [C.c_void_p] * 6, C.c_int),
    "kl_rmsnorm_fwd_b": ([C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong,
                          C.c_void_p, C.c_longlong, C.c_void_p], C.c_int),
    "kl_rmsnorm_bwd_b": ([C.c_int, C.c_int, C.c_int, C.c_float, C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong,
                          C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong, C.c_int,
                          C.c_void_p], C.c_int),
    "kl_recent_rows_fwd": ([C.c_int] * 5 + [C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p], C.c_int),
    "kl_recent_rows_bwd": ([C.c_int] * 5 + [C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p, C.c_longlong, C.c_void_p], C.c_int),
    "kl_gram_triu_fwd": ([C.c_int] * 4 + [C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p, C.c_longlong, C.c_void_p], C.c_int),
    "kl_gram_triu_bwd": ([C.c_int] * 4 + [C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p, C.c_longlong,
                                          C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p], C.c_int),
    "kl_rowdot3": ([C.c_int] * 4 + [C.c_void_p, C.c_longlong, C.c_longlong, C.c_void_p, C.c_longlong, C.c_longlong,
                                   C.c_void_p, C.c_longlong, C.c_void_p], C.c_int),
    "kl_regroup": ([C.c_void_p, C.c_void_p], C.c_int),
    "kl_memset": ([C.c_void_p, C.c_longlong, C.c_void_p], C.c_int),
    "kl_rowdot": ([C.c_int] * 3 + [C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong, C.c_void_p, C.c_void_p],
                  C.c_int),
    "kl_gated_sum_fwd": ([C.c_int] * 3 + [C.c_void_p, C.c_longlong] + [C.c_void_p] * 5 + [C.c_longlong, C.c_void_p], C.c_int),
    "kl_gated_sum_bwd": ([C.c_int] * 3 + [C.c_void_p, C.c_longlong] + [C.c_void_p] * 10, C.c_int),
    "kl_bce_fwd_bwd": ([C.c_int] + [C.c_void_p] * 5, C.c_int),
    "kl_ne": ([C.c_int, C.c_int] + [C.c_void_p] * 4, C.c_int),
    "kl_rote": ([C.c_void_p, C.c_void_p], C.c_int),
    "kl_cast": ([C.c_longlong, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "kl_act_fwd": ([C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong, C.c_int, C.c_int,
                    C.c_void_p, C.c_void_p], C.c_int),
    "kl_act_bwd": ([C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_longlong, C.c_void_p, C.c_longlong, C.c_void_p,
                    C.c_longlong, C.c_int, C.c_int, C.c_void_p, C.c_void_p], C.c_int),
    "kl_adam_tick": ([C.c_void_p, C.c_void_p], C.c_int),
    "kl_adam_step": ([C.c_longlong, C.c_float, C.c_float, C.c_float, C.c_float, C.c_int] + [C.c_void_p] * 7,
                     C.c_int),
    "kl_check_finite": ([C.c_longlong, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p], C.c_int),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load the CUDA library (raises if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libkunlun_sm100a.so not built ({LIB_PATH}); run `make` or __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _check(rc: int, what: str) -> None:
    if rc == KL_OK:
        return
    msg = lib().kl_last_error().decode(errors="replace")
    if rc == KL_EBADSHAPE:
        raise ShapeError(f"{what}: {msg}")
    if rc == KL_EUNSUPPORTED:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what}: {msg}")


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _need_cuda(*ts) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise RuntimeError("kunlun CUDA ops need CUDA tensors (no CPU fallback)")


def dt(t: torch.Tensor) -> int:
    if t.dtype == torch.float32:
        return KL_F32
    if t.dtype == torch.bfloat16:
        return KL_BF16
    raise ValueError(f"unsupported dtype {t.dtype}")


def ptr(t):
    return None if t is None else t.data_ptr()


def _as4(t: torch.Tensor) -> torch.Tensor:
    while t.dim() < 4:
        t = t.unsqueeze(0)
    if t.dim() != 4:
        raise ShapeError(f"gemm operands have at most 2 batch dims, got shape {tuple(t.shape)}")
    return t


_WS = {}
WS_BYTES = 64 << 20  # split-K scratch per device (GEMMs run stream-ordered, so one buffer is reused)


def _workspace(device) -> torch.Tensor:
    """Split-K scratch, one per (device, stream): GEMMs of parallel stream /
    graph branches run concurrently and must not share it."""
    key = (device, torch.cuda.current_stream(device).cuda_stream)
    ws = _WS.get(key)
    if ws is None:
        ws = torch.empty(WS_BYTES // 4, dtype=torch.float32, device=device)
        _WS[key] = ws
    return ws


def _bstride(t: torch.Tensor, i: int) -> int:
    return 0 if t.shape[i] == 1 else t.stride(i)


def gemm(A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None, *, out_dtype=None,
         alpha: float = 1.0, beta: float = 0.0, bias: torch.Tensor | None = None, acts=None,
         act_group: int = 1, aux: torch.Tensor | None = None, aux_mode: int = 0,
         residual: torch.Tensor | None = None, row_limit: torch.Tensor | None = None,
         reduce=(False, False)) -> torch.Tensor:
    """out[z] = epi(A[z] @ B[z]) over up to two (broadcastable) batch dims.

    A (..., M, K), B (..., K, N) are arbitrary strided views; ``reduce[i]``
    sums batch dim i (of the 2 padded leading dims) into a single output.
    ``out`` (..., M, N) is written in place when given (``beta`` reads it).
    """
    _need_cuda(A, B, out, bias, residual, aux, row_limit)
    if A.dtype != B.dtype:
        raise ValueError(f"gemm operand dtypes differ: {A.dtype} vs {B.dtype}")
    A4, B4 = _as4(A), _as4(B)
    M, K = A4.shape[2], A4.shape[3]
    if B4.shape[2] != K:
        raise ShapeError(f"gemm inner dims differ: {tuple(A.shape)} @ {tuple(B.shape)}")
    N = B4.shape[3]
    nb1 = max(A4.shape[0], B4.shape[0])
    nb2 = max(A4.shape[1], B4.shape[1])
    for t4 in (A4, B4):
        if t4.shape[0] not in (1, nb1) or t4.shape[1] not in (1, nb2):
            raise ShapeError("gemm batch dims do not broadcast")
    red1, red2 = bool(reduce[0]), bool(reduce[1])
    oshape = (1 if red1 else nb1, 1 if red2 else nb2, M, N)
    if out is None:
        lead = max(A.dim(), B.dim()) - 2
        out = torch.empty(oshape[2 - lead:], device=A.device, dtype=out_dtype or A.dtype)
    ret = out
    O4 = _as4(out)
    if tuple(O4.shape[2:]) != (M, N):
        raise ShapeError(f"gemm output shape {tuple(out.shape)} != (.., {M}, {N})")
    if (SWAP_SMALL_M and A.dtype == torch.bfloat16 and M < 64 and N >= 2 * M and N >= 64 and bias is None
            and not acts and aux is None and row_limit is None):
        # Small-M product on the 128-row tcgen05 tile: compute C^T = B^T A^T so
        # the long dimension fills the MMA rows (element-wise epilogue only).
        R4 = _as4(residual).transpose(2, 3) if residual is not None else None
        gemm(B4.transpose(2, 3), A4.transpose(2, 3), O4.transpose(2, 3), alpha=alpha, beta=beta,
             residual=R4, reduce=reduce)
        return ret
    a = GemmArgs()
    a.M, a.N, a.K = M, N, K
    a.nb1, a.nb2, a.red1, a.red2 = nb1, nb2, int(red1), int(red2)
    a.ab_dtype, a.c_dtype = dt(A), dt(out)
    a.A = A4.data_ptr()
    a.a_rs, a.a_cs, a.a_s1, a.a_s2 = A4.stride(2), A4.stride(3), _bstride(A4, 0), _bstride(A4, 1)
    a.B = B4.data_ptr()
    a.b_rs, a.b_cs, a.b_s1, a.b_s2 = B4.stride(2), B4.stride(3), _bstride(B4, 0), _bstride(B4, 1)
    a.C = O4.data_ptr()
    a.c_rs, a.c_cs, a.c_s1, a.c_s2 = O4.stride(2), O4.stride(3), _bstride(O4, 0), _bstride(O4, 1)
    if residual is not None:
        R4 = _as4(residual)
        if residual.dtype != out.dtype:
            raise ValueError("residual dtype must equal the output dtype")
        a.R = R4.data_ptr()
        a.r_rs, a.r_cs, a.r_s1, a.r_s2 = R4.stride(2), R4.stride(3), _bstride(R4, 0), _bstride(R4, 1)
    if aux is not None:
        X4 = _as4(aux)
        if X4.stride() != O4.stride() or aux.dtype != out.dtype:
            raise ShapeError("aux must share the output's strides and dtype")
        a.aux = X4.data_ptr()
    a.aux_mode = aux_mode
    a.alpha, a.beta = alpha, beta
    if bias is not None:
        if bias.dtype != torch.float32 or not bias.is_contiguous():
            raise ValueError("bias must be contiguous fp32")
        a.bias = bias.data_ptr()
    if row_limit is not None:
        if row_limit.dtype != torch.int32:
            raise ValueError("row_limit must be int32")
        a.row_limit = row_limit.data_ptr()
    if acts:
        codes = [ACT_CODES[x] if isinstance(x, str) else int(x) for x in acts]
        if len(codes) > MAX_ACT:
            raise ValueError("too many activation groups")
        a.n_act = len(codes)
        a.act_group = act_group
        for i, c in enumerate(codes):
            a.act_codes[i] = c
    if GEMM_LOG is not None:
        torch.cuda.synchronize()  # isolate this GEMM: no host-issue gaps inside the window
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
    ws = _workspace(A.device)
    a.workspace, a.workspace_bytes = ws.data_ptr(), ws.numel() * 4
    if OP_LOG is not None:
        _logged("kl_gemm", f"{M}x{N}x{K} b{nb1}x{nb2} r{int(red1)}{int(red2)}", lib().kl_gemm, C.byref(a), _stream())
    elif WORK is not None:
        ea, ec = A.element_size(), out.element_size()
        nA = (A4.shape[0] * A4.shape[1]) * M * K
        nB = (B4.shape[0] * B4.shape[1]) * K * N
        nC = oshape[0] * oshape[1] * M * N
        nbytes = (nA + nB) * ea + nC * ec * (2 if beta != 0.0 else 1) + (nC * ec if residual is not None else 0) \
            + (nC * ec if aux is not None else 0)
        fam = "gemm"
        _check(_record_work(fam, 2.0 * M * N * K * nb1 * nb2, float(nbytes), lib().kl_gemm, C.byref(a), _stream()),
               "kl_gemm")
    else:
        _check(lib().kl_gemm(C.byref(a), _stream()), "kl_gemm")
    if GEMM_LOG is not None:
        e.record()
        import traceback

        site = [f"{os.path.basename(f.filename)}:{f.lineno}:{f.name}" for f in traceback.extract_stack(limit=4)[:-1]]
        GEMM_LOG.append(((M, N, K, nb1, nb2, int(red1), int(red2), (a.a_rs, a.a_cs), (a.b_rs, a.b_cs),
                          (a.c_rs, a.c_cs), a.c_dtype, a.aux_mode, int(bool(residual is not None)), len(acts or ()),
                          lib().kl_last_gemm_path(), "<".join(reversed(site))), s, e))
    return ret


SWAP_SMALL_M = False  # operand-swapped small-M form (measured slower than the plain tcgen05 tile: strided epilogue)
GEMM_LOG = None  # list of (M, N, K, nb1, nb2, red1, red2, A/B/C strides, c_dtype, path) when set


def swa_args(qkv, lengths, H, d_h, w, causal, O, LSE, dO=None, dqkv=None, Dbuf=None) -> SwaArgs:
    B, T = qkv.shape[0], qkv.shape[1]
    a = SwaArgs()
    a.B, a.T, a.H, a.d_h, a.w, a.causal = B, T, H, d_h, int(w), int(causal)
    a.dtype = dt(qkv)
    a.scale = 1.0 / float(d_h) ** 0.5
    a.lengths = lengths.data_ptr()
    a.QKV, a.ld_qkv, a.bs_qkv = qkv.data_ptr(), qkv.stride(1), qkv.stride(0)
    a.O, a.ld_o, a.bs_o = O.data_ptr(), O.stride(1), O.stride(0)
    a.LSE = LSE.data_ptr()
    if dO is not None:
        if dO.stride() != O.stride():
            raise ShapeError("dO must share O's strides")
        a.dO = dO.data_ptr()
        a.dQKV = dqkv.data_ptr()
        a.Dbuf = Dbuf.data_ptr()
    return a


TIMED = None  # {entry-point name: [(start, end) CUDA events]} while bench.py times ops
TIMED_EXTERNAL = False  # record event nodes that survive CUDA-graph capture


OP_LOG = None  # list of (entry, shape, call site, ms) while bench.py --op-census runs one eager step


def _site() -> str:
    import traceback

    fr = [f for f in traceback.extract_stack()[:-3] if "paper_2602_10016_b200" in f.filename
          and not f.filename.endswith("_capi.py")]
    return "<".join(f"{os.path.basename(f.filename)[:-3]}:{f.name}:{f.lineno}" for f in reversed(fr[-3:]))


def _logged(name, shape, fn, *args):
    """Times one C-ABI call alone on the device (synchronize on both sides)."""
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200000)  # keeps the device busy while the host prepares the launch
    s.record()
    n0 = launch_count()
    rc = fn(*args)
    e.record()
    e.synchronize()
    OP_LOG.append((name, shape, _site(), s.elapsed_time(e), launch_count() - n0))
    _check(rc, name)


# Per-launch work accounting for bench.py's roofline table: while WORK is a
# list, every accounted entry point records (family, algorithmic flops,
# algorithmic bytes, start event, end event) around its launch on the
# launching stream (external events survive CUDA-graph capture, so a captured
# step's replays refresh the durations).
WORK = None


def _support_total(T, w, causal):
    import numpy as np

    i = np.arange(T)
    hi = np.minimum(i + w, T - 1) if not causal else i
    return int((hi - np.maximum(i - w, 0) + 1).sum())


def _work_of(name, args):
    """(family, flops, bytes) of one launch from its C-ABI arguments (the
    algorithmic work: operands read once, results written once)."""
    a = args[0]._obj if args and hasattr(args[0], "_obj") else None
    if name in ("kl_swa_fwd", "kl_swa_bwd") and a is not None:
        HD = a.H * a.d_h
        sup = _support_total(a.T, a.w, bool(a.causal))
        if name == "kl_swa_fwd":
            return "swa_fwd", 4.0 * sup * HD * a.B, float(a.B) * a.T * (3 * HD * 2 + HD * 2 + a.H * 4)
        return "swa_bwd", 10.0 * sup * HD * a.B, float(a.B) * a.T * (3 * HD * 2 * 2 + HD * 2 * 2 + a.H * 4 * 2)
    if name in ("kl_gdpa_fwd", "kl_gdpa_bwd") and a is not None:
        mm = 2.0 * a.B * a.T * a.HK * a.d
        kv = 2.0 * a.B * a.HK * a.d * 2
        if name == "kl_gdpa_fwd":
            return "gdpa_fwd", 2 * mm, 2.0 * a.B * a.T * a.d * 2 + kv
        return "gdpa_bwd", 5 * mm, 3.0 * a.B * a.T * a.d * 2 + 2 * kv
    if name in ("kl_hsp_fwd", "kl_hsp_bwd") and a is not None:
        mm = 2.0 * a.B * a.T * a.HQ * a.d
        if name == "kl_hsp_fwd":
            return "hsp_fwd", 2 * mm, float(a.B) * a.T * a.d * 2
        return "hsp_bwd", 4 * mm, 2.0 * a.B * a.T * a.d * 2 + 2.0 * a.B * a.HQ * a.T * 2 * 2
    if name in ("kl_colsoftmax_fwd", "kl_colsoftmax_bwd") and a is not None:
        n = float(a.Bn) * a.T * a.C
        return ("colsoftmax_fwd", 0.0, n * 6) if name == "kl_colsoftmax_fwd" else ("colsoftmax_bwd", 0.0, n * 12)
    if name == "kl_adam_step":
        return "adam", 0.0, float(args[0]) * 30  # fp32 p, g, m, v read; p, m, v + bf16 mirror written
    return None


WORK_EVENTS = True  # False: log the work only (durations come from a profiler pass)


def _record_work(fam, flops, nbytes, fn, *args):
    if not WORK_EVENTS:
        WORK.append((fam, flops, nbytes, None, None))
        return fn(*args)
    s = torch.cuda.Event(enable_timing=True, external=True)
    e = torch.cuda.Event(enable_timing=True, external=True)
    s.record()
    rc = fn(*args)
    e.record()
    WORK.append((fam, flops, nbytes, s, e))
    return rc


def call(name: str, *args):
    if WORK is not None:
        w = _work_of(name, args)
        if w is not None:
            _check(_record_work(w[0], w[1], w[2], getattr(lib(), name), *args), name)
            return
    if OP_LOG is not None:
        _logged(name, "", getattr(lib(), name), *args)
        return
    if TIMED is not None and name in TIMED:
        s = torch.cuda.Event(enable_timing=True, external=TIMED_EXTERNAL)
        e = torch.cuda.Event(enable_timing=True, external=TIMED_EXTERNAL)
        s.record()
        rc = getattr(lib(), name)(*args)
        e.record()
        TIMED[name].append((s, e))
        _check(rc, name)
        return
    _check(getattr(lib(), name)(*args), name)


def launch_count() -> int:
    return int(lib().kl_launch_count())


# Kernel-path counters (include/kunlun_capi.h KL_PATH_*).
PATHS = {"gemm_tc": 0, "gemm_simt": 1, "gdpa_fwd_tc": 2, "gdpa_bwd_tc": 3, "hsp_fwd_tc": 4, "hsp_bwd_tc": 5,
         "swa_fwd_tc": 6, "swa_bwd_tc": 7, "swa_fwd_simt": 8, "swa_bwd_simt": 9, "colsoftmax": 10,
         "gdpa_fwd_tc512": 11, "gdpa_bwd_tc512": 12, "hsp_fwd_split": 13, "gemm_wide": 14}


def path_hits() -> dict:
    """{kernel family: launches since load / the last reset_path_hits()}."""
    L = lib()
    return {k: int(L.kl_path_hits(v)) for k, v in PATHS.items()}


def reset_path_hits() -> None:
    lib().kl_reset_path_hits()
