"""Differentiable device ops of the Kunlun hot path.

Each ``torch.autograd.Function`` here is the B200 analogue of the reference's
``record(out, parents, vjp)`` plugin hook (tensor.py:185-195): forward and
VJP both run hand-written sm_100a kernels from libkunlun_sm100a.so via the C
ABI (``_capi``).  There is no CPU or library fallback.

Parameters are not autograd leaves one by one: they live in the flat
``Params`` buffer, kernels read the compute-dtype mirror and the backward
kernels *accumulate* fp32 weight gradients straight into ``Params.gflat``
(beta=1 epilogues).  Every parameter-consuming Function takes
``Params.flat`` (requires_grad) as a dummy input so autograd always runs its
backward.
"""

from __future__ import annotations

import ctypes as C

import os

import torch

from . import _capi
from ._capi import gemm
from .tensor import ACTIVATIONS, ShapeError, flag_nonfinite, numerics_check_mode


class PRef:
    """A parameter operand: block ``key`` of ``P`` seen through ``fn``."""

    __slots__ = ("P", "key", "fn", "fp32")

    def __init__(self, P, key, fn=None, fp32=False):
        self.P, self.key, self.fn, self.fp32 = P, key, fn, fp32

    def w(self):
        v = self.P.w32(self.key) if self.fp32 else self.P.w(self.key)
        return self.fn(v) if self.fn else v

    def g(self):
        v = self.P.g(self.key)
        return self.fn(v) if self.fn else v


class SRef(PRef):
    """A stacked parameter operand: blocks ``keys`` (one per grouped event
    type, equally shaped and uniformly spaced in the flat buffers) seen as one
    (G, ...) tensor through ``fn`` (Params.stacked)."""

    __slots__ = ("keys",)

    def __init__(self, P, keys, fn=None, fp32=False):
        super().__init__(P, keys[0], fn, fp32)
        self.keys = tuple(keys)

    def w(self):
        v = self.P.stacked(self.keys, "w32" if self.fp32 else "w")
        return self.fn(v) if self.fn else v

    def g(self):
        v = self.P.stacked(self.keys, "g")
        return self.fn(v) if self.fn else v


class GradSink:
    """One gradient buffer shared by the consumers of a (B, T, d) sequence
    tensor inside a layer (HSP pooling + recent rows, the GDPA / attention
    branch), delivered to autograd by ONE ``_SeqJoin`` node.

    The layer applies ``seq_join(S, sink)`` once and hands its output to the
    consumers.  The first consumer whose backward runs registers its dS
    (``put``); later consumers accumulate into it — the fused HSP kernel in
    its own epilogue (``take`` + accumulate_ds), others with one add — and
    every participating consumer returns *no* gradient for S.  The join's
    backward then returns the buffer: autograd never materialises one
    (B, T, d) gradient per consumer and never adds them.  Consumers outside
    the layer (a caller reading the layer output) see S itself, not the
    join's output, so autograd sums their gradients with the join's buffer —
    correct for any graph, not just the model's own.

    The consumers may run on different streams (parallel branches): ``take``
    orders the accumulation after the registering stream's write,
    ``release`` orders the registering stream's later work after it, and the
    join waits for the registering stream."""

    __slots__ = ("t", "stream")

    def __init__(self):
        self.t = None
        self.stream = None

    def put(self, t):
        self.t = t
        self.stream = torch.cuda.current_stream(t.device) if t.is_cuda else None

    def take(self, like):
        t = self.t
        if t is not None and t.shape == like.shape and t.dtype == like.dtype and t.is_contiguous():
            if self.stream is not None:
                cur = torch.cuda.current_stream(t.device)
                if cur != self.stream:
                    cur.wait_stream(self.stream)
                    t.record_stream(cur)
            return t
        return None

    def release(self):
        if self.stream is not None:
            cur = torch.cuda.current_stream(self.t.device)
            if cur != self.stream:
                self.stream.wait_stream(cur)

    def deliver(self, dS):
        """A consumer's backward hands over its full dS: registered if it is
        the first, else added into the registered buffer.  Returns the
        gradient the consumer must return to autograd (always None)."""
        if self.t is None:
            self.put(dS)
        else:
            acc = self.take(dS)
            if acc is None:
                raise ShapeError("shared sequence gradient: shape / dtype mismatch")
            acc.add_(dS)
            self.release()
        return None


class _SeqJoin(torch.autograd.Function):
    """Identity whose output feeds a layer's sequence consumers; its
    backward returns the GradSink buffer they filled (plus, if some
    consumer returned an ordinary gradient, that gradient)."""

    @staticmethod
    def forward(ctx, S, sink):
        ctx.sink = sink
        ctx.set_materialize_grads(False)
        return S.view_as(S)

    @staticmethod
    def backward(ctx, g):
        sink = ctx.sink
        t = sink.t
        sink.t = None
        if t is None:
            return g, None
        if sink.stream is not None:
            cur = torch.cuda.current_stream(t.device)
            if cur != sink.stream:
                cur.wait_stream(sink.stream)
                t.record_stream(cur)
        return (t if g is None else t + g), None


def seq_join(S, sink):
    """S for a layer's sequence consumers that share ``sink`` (GradSink)."""
    return _SeqJoin.apply(S, sink)


class ResidualStash:
    """Passes the residual gradient of a later op (out-projection: y = S + o
    W^T) to an earlier op with the same input (the QKV projection), which
    adds it in its dX GEMM epilogue: backward of the later op always runs
    first (the earlier op's output gradient depends on it)."""

    __slots__ = ("g",)

    def __init__(self):
        self.g = None


def _codes(acts):
    if acts is None:
        return []
    if isinstance(acts, str):
        acts = [acts]
    return [ACTIVATIONS[a] for a in acts]


def _stream():
    return _capi._stream()


_SIDE = {}
BRANCH_STREAMS = os.environ.get("KL_BRANCH_STREAMS", "1") != "0"


def side_streams(device):
    """Every side stream created so far on ``device``."""
    idx = torch.device(device).index or 0
    return [st for (i, _), st in _SIDE.items() if i == idx]


def side_stream(device, name="side"):
    """Cached side streams per (device, name) for independent branches
    (distinct names for nested branch sets)."""
    key = (torch.device(device).index or 0, name)
    if key not in _SIDE:
        _SIDE[key] = torch.cuda.Stream(device=device)
    return _SIDE[key]


# Weight gradients on their own stream: while a training step runs
# (optim.TrainStep sets DW_STREAM), every weight / bias gradient GEMM is issued
# on a "dw" side stream (forked from the node's stream), so the long-K,
# HBM-bound dW products overlap the activation-gradient chain; TrainStep joins
# the stream before the optimizer.  Off by default: a bare loss.backward()
# leaves every kernel on the caller's streams.
DW_STREAM = False
DW_STREAM_FWD = False  # set by TrainStep around its forward (query folds on the summary-branch stream)


class _DwFork:
    __slots__ = ("prev", "st", "on")

    def __init__(self, tensors):
        self.on = DW_STREAM and torch.cuda.is_available()
        if self.on:
            dev = next(t.device for t in tensors if isinstance(t, torch.Tensor))
            cur = torch.cuda.current_stream(dev)
            self.st = side_stream(dev, "dw")
            self.st.wait_stream(cur)
            for t in tensors:
                if isinstance(t, torch.Tensor):
                    t.record_stream(self.st)

    def __enter__(self):
        if self.on:
            self.prev = torch.cuda.current_stream(self.st.device)
            torch.cuda.set_stream(self.st)
        return self

    def __exit__(self, *exc):
        if self.on:
            torch.cuda.set_stream(self.prev)
        return False


def dw_join(device):
    """Current stream waits for every side stream (weight gradients, branch
    work whose results autograd does not see, e.g. in-place parameter
    gradients written on a branch stream)."""
    if torch.cuda.is_available():
        cur = torch.cuda.current_stream(device)
        side_stream(device, "dw")
        for st in side_streams(device):
            if st != cur:
                cur.wait_stream(st)


def run_branches(fns, device, inputs=(), name="side", side_first=False):
    """Run independent branches ``fns`` (callables) alternately on the current
    and a side stream, joined before returning; inside a CUDA graph capture
    this becomes a fork / join of parallel graph branches, so the branches'
    small kernels overlap.  Autograd runs each branch's backward on the stream
    its forward ran on, so the backward branches overlap the same way.
    Tensors crossing streams are recorded on the consuming stream."""
    if not BRANCH_STREAMS or len(fns) < 2 or not torch.cuda.is_available():
        return [f() for f in fns]
    main = torch.cuda.current_stream(device)
    side = side_stream(device, name)
    side.wait_stream(main)
    for t in inputs:  # made on the current stream, read by the side branches
        if isinstance(t, torch.Tensor):
            t.record_stream(side)
    outs = []
    # side_first: even-indexed branches go to the side stream.  The branch
    # issued last creates the newest autograd nodes, whose backward runs
    # first; callers use this to pick which branch's backward leads.
    on_side = [(i % 2 == 0) == side_first for i in range(len(fns))]
    for i, f in enumerate(fns):
        st = side if on_side[i] else main
        with torch.cuda.stream(st):
            outs.append(f())
    main.wait_stream(side)

    def record(o):
        if isinstance(o, torch.Tensor):
            o.record_stream(main)
        elif isinstance(o, (list, tuple)):
            for x in o:
                record(x)

    for i, o in enumerate(outs):
        if on_side[i]:
            record(o)
    return outs


def _as4(t):
    while t.dim() < 4:
        t = t.unsqueeze(0)
    return t


def _bcast_reduce(op4, out4):
    """Batch dims where an operand was broadcast against the output."""
    return (op4.shape[0] == 1 and out4.shape[0] > 1, op4.shape[1] == 1 and out4.shape[1] > 1)


# ---------------------------------------------------------------------------
class _MM(torch.autograd.Function):
    """C = alpha * A @ B (+ residual) over up to two broadcast batch dims,
    optionally summing batch dims (``reduce``).  Operands are tensors or
    parameter references.  VJP: dA = g B^T, dB = A^T g (tensor.py:283-289),
    reducing over batch dims where an operand was broadcast."""

    @staticmethod
    def forward(ctx, a, b, flat, aref, bref, reduce, alpha, residual):
        A = aref.w() if aref is not None else a
        Bm = bref.w() if bref is not None else b
        out = gemm(A, Bm, alpha=alpha, reduce=reduce, residual=residual)
        ctx.aref, ctx.bref, ctx.alpha = aref, bref, alpha
        ctx.has_res = residual is not None
        ctx.save_for_backward(a if aref is None else None, b if bref is None else None)
        ctx.ashape = tuple(A.shape)
        ctx.bshape = tuple(Bm.shape)
        return out

    @staticmethod
    def backward(ctx, g):
        a_t, b_t = ctx.saved_tensors
        A = ctx.aref.w() if ctx.aref is not None else a_t
        Bm = ctx.bref.w() if ctx.bref is not None else b_t
        g4 = _as4(g)
        nb = (max(_as4(A).shape[0], _as4(Bm).shape[0]), max(_as4(A).shape[1], _as4(Bm).shape[1]))
        g4 = g4.expand(nb[0], nb[1], g4.shape[2], g4.shape[3])
        da = db = None
        A4, B4 = _as4(A), _as4(Bm)
        if ctx.aref is not None or ctx.needs_input_grad[0]:
            red = _bcast_reduce(A4, g4)
            if ctx.aref is not None:
                with _DwFork((g, Bm)):
                    gemm(g4, B4.transpose(2, 3), _as4(ctx.aref.g()), alpha=ctx.alpha, beta=1.0, reduce=red)
            else:
                da = gemm(g4, B4.transpose(2, 3), alpha=ctx.alpha, reduce=red)
                da = da.reshape(a_t.shape)
        if ctx.bref is not None or ctx.needs_input_grad[1]:
            red = _bcast_reduce(B4, g4)
            if ctx.bref is not None:
                with _DwFork((g, A)):
                    gemm(A4.transpose(2, 3), g4, _as4(ctx.bref.g()), alpha=ctx.alpha, beta=1.0, reduce=red)
            else:
                db = gemm(A4.transpose(2, 3), g4, alpha=ctx.alpha, reduce=red)
                db = db.reshape(b_t.shape)
        dres = g if ctx.has_res else None
        return da, db, None, None, None, None, None, dres


def mm(a, b, P=None, *, reduce=(False, False), alpha=1.0, residual=None):
    """Batched matmul of tensors / ``PRef`` parameters (see ``_MM``)."""
    aref = a if isinstance(a, PRef) else None
    bref = b if isinstance(b, PRef) else None
    P = P or (aref.P if aref else (bref.P if bref else None))
    flat = P.flat if P is not None else None
    return _MM.apply(None if aref else a, None if bref else b, flat, aref, bref, tuple(reduce), float(alpha),
                     residual)


# ---------------------------------------------------------------------------
class _Linear(torch.autograd.Function):
    """y = act(x W^T + b) + residual; W (N, K) in the reference (out, in)
    layout (mlp.py:47-59, attention projections).  Saves the pre-activation
    (epilogue aux) for the VJP."""

    @staticmethod
    def forward(ctx, x, flat, P, wkey, bkey, act, residual, out_dtype=None, stash_out=None, stash_in=None):
        W = _pw(P, wkey)
        N = W.shape[-2]
        codes = _codes(act) if act and act != "identity" else []
        pre = None
        bias = P.w32(bkey) if bkey else None
        x4 = x if x.dim() >= 2 else x.unsqueeze(0)
        if codes:
            pre = torch.empty(x4.shape[:-1] + (N,), device=x.device, dtype=x.dtype)
        y = gemm(x4, W.transpose(-1, -2), bias=bias, acts=codes or None, aux=pre, aux_mode=1 if codes else 0,
                 residual=residual, out_dtype=out_dtype)
        ctx.P, ctx.wkey, ctx.bkey, ctx.codes = P, wkey, bkey, codes
        ctx.has_res = residual is not None
        ctx.xshape = x.shape
        ctx.stash_out, ctx.stash_in = stash_out, stash_in
        ctx.save_for_backward(x4, pre)
        return y if x.dim() >= 2 else y.squeeze(0)

    @staticmethod
    def backward(ctx, g):
        x4, pre = ctx.saved_tensors
        P = ctx.P
        W = _pw(P, ctx.wkey)
        g = g.contiguous()
        if g.dtype != W.dtype:  # fp32-output linear (weight generation)
            g = cast(g, W.dtype)
        if g.dim() < x4.dim():
            g = g.unsqueeze(0)
        gp = g
        if ctx.codes:
            gp = torch.empty_like(g)
            cols = g.shape[-1]
            rows = g.numel() // cols
            codes = (C.c_int * len(ctx.codes))(*ctx.codes)
            _capi.call("kl_act_bwd", rows, cols, _capi.dt(g), g.data_ptr(), cols, pre.data_ptr(), cols,
                       gp.data_ptr(), cols, len(ctx.codes), 1, codes, _stream())
        dx = None
        if ctx.needs_input_grad[0]:
            res = None
            if ctx.stash_in is not None and ctx.stash_in.g is not None:
                res = ctx.stash_in.g  # a later op's residual gradient for the same input
                ctx.stash_in.g = None
                res = res.reshape(gp.shape[:-1] + (res.shape[-1],))
            dx = gemm(gp, W, residual=res)
            dx = dx.reshape(ctx.xshape)
        # dW = sum over rows (and batch dims) of gp^T x
        gp4, x44 = _as4(gp), _as4(x4)
        rows = gp.numel() // gp.shape[-1]
        gpc = gp if gp.is_contiguous() else gp.contiguous()
        ones = _ones(rows, gp.dtype, gp.device) if ctx.bkey else None
        grouped = not isinstance(ctx.wkey, str)  # one weight per group (leading batch dim): no reduction over it
        with _DwFork((gp, gpc, x4, ones)):
            gemm(gp4.transpose(2, 3), x44, _as4(_pg(P, ctx.wkey)) if grouped else P.g(ctx.wkey), beta=1.0,
                 reduce=(True, not grouped))
            if ctx.bkey:
                gemm(ones.view(1, rows), gpc.view(rows, -1), P.g(ctx.bkey).view(1, -1), beta=1.0)
        dres = g.reshape(ctx.xshape[:-1] + (g.shape[-1],)) if ctx.has_res else None
        if dres is not None and ctx.stash_out is not None:
            ctx.stash_out.g = dres  # added by the earlier op's dX epilogue instead
            dres = None
        return dx, None, None, None, None, None, dres, None, None, None


_ONES = {}


def _ones(n, dtype, device):
    key = (dtype, device)
    t = _ONES.get(key)
    if t is None or t.numel() < n:
        t = torch.ones(max(n, 1024), dtype=dtype, device=device)
        _ONES[key] = t
    return t[:n]


def _pw(P, key):
    """A weight block, or (a tuple of keys) the (G, ...) stack of equally
    shaped, uniformly spaced blocks (grouped event types; Params.stacked)."""
    return P.w(key) if isinstance(key, str) else P.stacked(key, "w")


def _pg(P, key):
    return P.g(key) if isinstance(key, str) else P.stacked(key, "g")


def linear(x, P, wkey, bkey=None, act=None, residual=None, out_dtype=None, stash_out=None, stash_in=None):
    """y = act(x W^T + b) + residual.  ``stash_out`` / ``stash_in``: a
    ResidualStash shared with an earlier linear on the same input.  A tuple
    ``wkey`` is a grouped linear: x (G, M, K) with one stacked weight per
    group (Params.stacked), no bias."""
    if not isinstance(wkey, str) and bkey is not None:
        raise ValueError("grouped linear takes no bias")
    return _Linear.apply(x, P.flat, P, wkey, bkey, act, residual, out_dtype, stash_out, stash_in)



# ---------------------------------------------------------------------------
class _GdpaCore(torch.autograd.Function):
    """Folded GDPA core per sample (gdpa.py:120-187):
        Z = S Kt^T / tau,  A = Act_h(Z) (per n_kv column block),
        Y = S + A Vt;   rows >= length pass through (Y = S).
    VJP: dZ = (G Vt^T) * Act'(Z) / tau, dS = G + dZ Kt, dKt = dZ^T S, dVt = A^T G.

    bf16 with H*n_kv = 64 and d in {128, 256} runs the fused tcgen05 kernels
    kl_gdpa_fwd / kl_gdpa_bwd (Z and A stay on chip, recomputed in the
    backward); every other case composes kl_gemm calls with fused epilogues
    (the fp32 parity path)."""

    @staticmethod
    def forward(ctx, S, Kt, Vt, lengths, codes, n_kv, inv_tau, sink=None):
        B, T, d = S.shape
        HK = Kt.shape[1]
        ctx.codes, ctx.n_kv, ctx.inv_tau, ctx.sink = codes, n_kv, inv_tau, sink
        ctx.fused = _gdpa_fused_ok(S, HK, codes, n_kv)
        if ctx.fused:
            S = S.contiguous()
            Kt, Vt = Kt.contiguous(), Vt.contiguous()
            Y = torch.empty_like(S)
            a = _gdpa_args(S, Kt, Vt, lengths, codes, n_kv, inv_tau)
            a.Y = Y.data_ptr()
            _capi.call("kl_gdpa_fwd", C.byref(a), _stream())
            ctx.save_for_backward(S, Kt, Vt, lengths)
            return Y
        Z = torch.empty(B, T, HK, device=S.device, dtype=S.dtype)
        A = torch.empty_like(Z)
        gemm(S, Kt.transpose(1, 2), A, alpha=inv_tau, acts=codes, act_group=n_kv, aux=Z, aux_mode=1,
             row_limit=lengths)
        Y = gemm(A, Vt, residual=S)
        ctx.save_for_backward(S, Kt, Vt, Z, A, lengths)
        return Y

    @staticmethod
    def backward(ctx, g):
        g = g.contiguous()
        if ctx.fused:
            S, Kt, Vt, lengths = ctx.saved_tensors
            dS = torch.empty_like(S)
            a = _gdpa_args(S, Kt, Vt, lengths, ctx.codes, ctx.n_kv, ctx.inv_tau)
            if S.shape[-1] == 512:
                # d = 512: the kernel forms dS and writes dZ, A (B, T, HK); the
                # sample-wide reductions dKt = dZ^T S, dVt = A^T dY are GEMMs
                B, T, _ = S.shape
                dZ = torch.empty(B, T, Kt.shape[1], device=S.device, dtype=S.dtype)
                A = torch.empty_like(dZ)
                a.dY, a.dS, a.dZ_out, a.A_out = g.data_ptr(), dS.data_ptr(), dZ.data_ptr(), A.data_ptr()
                _capi.call("kl_gdpa_bwd", C.byref(a), _stream())
                dKt = gemm(dZ.transpose(1, 2), S)
                dVt = gemm(A.transpose(1, 2), g)
            else:
                dKt, dVt = torch.empty_like(Kt), torch.empty_like(Vt)
                a.dY, a.dS, a.dKt, a.dVt = g.data_ptr(), dS.data_ptr(), dKt.data_ptr(), dVt.data_ptr()
                _capi.call("kl_gdpa_bwd", C.byref(a), _stream())
            if ctx.sink is not None:
                dS = ctx.sink.deliver(dS)
            return dS, dKt, dVt, None, None, None, None, None
        S, Kt, Vt, Z, A, lengths = ctx.saved_tensors
        dZ = torch.empty_like(Z)
        gemm(g, Vt.transpose(1, 2), dZ, alpha=ctx.inv_tau, acts=ctx.codes, act_group=ctx.n_kv, aux=Z, aux_mode=2,
             row_limit=lengths)
        dS = gemm(dZ, Kt, residual=g)
        dKt = gemm(dZ.transpose(1, 2), S)
        dVt = gemm(A.transpose(1, 2), g)
        if ctx.sink is not None:
            dS = ctx.sink.deliver(dS)
        return dS, dKt, dVt, None, None, None, None, None


GDPA_FUSED = True  # tests flip this to A/B the fused kernels against the GEMM composition


_FUSED_ACTS = tuple(ACTIVATIONS[a] for a in ("identity", "relu", "silu", "tanh"))


def _gdpa_fused_ok(S, HK, codes=(), n_kv=16) -> bool:
    """The fused kernels: bf16, (64 generated rows, d in {128, 256}) or
    (128 generated rows, d = 512), n_kv a multiple of 16, the default
    activation cycle (kl_gdpa_fwd's contract)."""
    d = S.shape[-1]
    return (GDPA_FUSED and S.dtype == torch.bfloat16 and ((HK == 64 and d in (128, 256)) or (HK == 128 and d == 512))
            and n_kv % 16 == 0 and all(c in _FUSED_ACTS for c in codes)
            and bool(_capi.lib().kl_tcgen05_available()))


def _gdpa_args(S, Kt, Vt, lengths, codes, n_kv, inv_tau):
    a = _capi.GdpaArgs()
    a.B, a.T, a.d = S.shape
    a.HK, a.n_kv = Kt.shape[1], n_kv
    a.dtype = _capi.dt(S)
    a.inv_tau = inv_tau
    a.n_act = len(codes)
    for i, c in enumerate(codes):
        a.act_codes[i] = c
    a.lengths = lengths.data_ptr()
    a.S, a.s_rs, a.s_bs = S.data_ptr(), S.stride(1), S.stride(0)
    a.Kt, a.Vt = Kt.data_ptr(), Vt.data_ptr()
    return a


def gdpa_core(S, Kt, Vt, lengths, acts, n_kv, inv_tau, sink=None):
    return _GdpaCore.apply(S, Kt, Vt, lengths, _codes(acts), int(n_kv), float(inv_tau), sink)


# ---------------------------------------------------------------------------
class _SwaCore(torch.autograd.Function):
    """Banded flash attention core (attention.py:69-129); QKV packed."""

    @staticmethod
    def forward(ctx, qkv, lengths, H, d_h, w, causal):
        B, T, _ = qkv.shape
        O = torch.empty(B, T, H * d_h, device=qkv.device, dtype=qkv.dtype)
        LSE = torch.empty(B, H, T, device=qkv.device, dtype=torch.float32)
        a = _capi.swa_args(qkv, lengths, H, d_h, w, causal, O, LSE)
        _capi.call("kl_swa_fwd", C.byref(a), _stream())
        ctx.save_for_backward(qkv, lengths, O, LSE)
        ctx.cfg = (H, d_h, w, causal)
        return O

    @staticmethod
    def backward(ctx, g):
        qkv, lengths, O, LSE = ctx.saved_tensors
        H, d_h, w, causal = ctx.cfg
        g = g.contiguous()
        dqkv = torch.empty_like(qkv)
        Dbuf = torch.empty_like(LSE)
        a = _capi.swa_args(qkv, lengths, H, d_h, w, causal, O, LSE, g, dqkv, Dbuf)
        _capi.call("kl_swa_bwd", C.byref(a), _stream())
        return dqkv, None, None, None, None, None


def swa_core(qkv, lengths, H, d_h, w, causal=False):
    if not qkv.is_contiguous():
        qkv = qkv.contiguous()
    return _SwaCore.apply(qkv, lengths, int(H), int(d_h), int(w), bool(causal))


# ---------------------------------------------------------------------------
def _colsm_args(X, P, lengths, LSE=None):
    a = _capi.ColSoftmaxArgs()
    a.Bn, a.T, a.C = X.shape[0], X.shape[1], X.shape[2]
    a.dtype_in, a.dtype_out = _capi.dt(X), _capi.dt(P)
    a.X, a.x_rs, a.x_bs = X.data_ptr(), X.stride(1), X.stride(0)
    a.P, a.p_rs, a.p_bs = P.data_ptr(), P.stride(1), P.stride(0)
    a.LSE = LSE.data_ptr() if LSE is not None else None
    a.lengths = lengths.data_ptr()
    return a


class _HspPool(torch.autograd.Function):
    """Seed/CLS-query cross-attention pooling with keys = values = S
    (hsp_seed_attend / pma, seqsum.py:26-34, 96-102, reassociated as
    P = softmax_t(S Q^T), pooled = P^T S — SURVEY.md §7.3 item 7).
    Q (HQ, d) is batch-shared, pre-scaled by 1/sqrt(d_h), rows ordered
    (query, head) so every pooled output (B, n, H, d) flattens to rows
    (b, query) with one stride.  ``splits`` cuts the HQ query rows into
    separately stored outputs (seed set, CLS set).  Length-0 samples pool to
    zeros with no gradient (seqsum.py:32-33, 99-100)."""

    @staticmethod
    def forward(ctx, S, Q32, lengths, splits, n_recent=0, sink=None):
        # Q arrives in fp32 (the batch-shared query path is computed in fp32);
        # the T-length work runs in S's dtype and dQ is returned in fp32.
        B, T, d = S.shape
        HQ = Q32.shape[-2]
        G = Q32.shape[0] if Q32.dim() == 3 else 1  # grouped event types: one query set per B / G samples
        if B % G:
            raise ShapeError(f"{G} query sets do not divide the batch of {B}")
        if sum(splits) != HQ:
            raise ShapeError(f"query splits {splits} do not cover {HQ} rows")
        Q = Q32
        if Q32.dtype != S.dtype:
            Q = torch.empty(Q32.shape, device=S.device, dtype=S.dtype)
            _capi.call("kl_cast", Q.numel(), _capi.dt(Q32), Q32.contiguous().data_ptr(), _capi.dt(Q), Q.data_ptr(),
                       _stream())
        ctx.splits = tuple(splits)
        ctx.n_recent, ctx.sink = n_recent, sink
        ctx.fused = _hsp_fused_ok(S, HQ, len(splits))
        rec = _recent_fwd(S, lengths, n_recent) if n_recent > 0 else None
        if ctx.fused:
            S = S.contiguous()
            outs = [torch.empty(B, n, d, device=S.device, dtype=S.dtype) for n in splits]
            LSE = torch.empty(B, HQ, device=S.device, dtype=torch.float32)
            a = _hsp_args(S, Q, lengths, splits[0], outs[0], outs[-1], LSE)
            ws = None
            if d == 512 and HSP_BALANCED:  # key blocks split over the SMs: per-part partials + arrival counters
                nb = int(_capi.lib().kl_hsp_fwd_workspace_bytes(C.byref(a)))
                ws = torch.empty(nb, device=S.device, dtype=torch.uint8)
                a.workspace, a.workspace_bytes = ws.data_ptr(), nb
            _capi.call("kl_hsp_fwd", C.byref(a), _stream())
            del ws
            ctx.save_for_backward(S, Q, lengths, LSE, *outs)
            return tuple(outs) + ((rec,) if rec is not None else ())
        sc = gemm(S.view(G, B // G, T, d), Q.view(G, 1, HQ, d).transpose(2, 3), out_dtype=torch.float32)
        sc = sc.view(B, T, HQ)
        Pm = torch.empty(B, T, HQ, device=S.device, dtype=S.dtype)
        lse = torch.empty(B, HQ, device=S.device, dtype=torch.float32)
        a = _colsm_args(sc, Pm, lengths, lse)
        _capi.call("kl_colsoftmax_fwd", C.byref(a), _stream())
        outs, c0 = [], 0
        for n in splits:
            outs.append(gemm(Pm[:, :, c0:c0 + n].transpose(1, 2), S))  # (B, n, d)
            c0 += n
        # the backward recomputes P in fp32 from the scores + LSE (a bf16 P
        # would feed its rounding into the cancellation-heavy dQ reduction)
        ctx.save_for_backward(S, Q, lengths, Pm, sc, lse, *outs)
        return tuple(outs) + ((rec,) if rec is not None else ())

    @staticmethod
    def backward(ctx, *gs):
        g_rec = None
        if ctx.n_recent > 0:
            gs, g_rec = gs[:-1], gs[-1]
        if ctx.fused:
            dS, dQ = _hsp_fused_bwd(ctx, gs)
        else:
            dS, dQ = _hsp_gemm_bwd(ctx, gs)
        if g_rec is not None:
            _recent_bwd_into(dS, g_rec, ctx.saved_tensors[2])
        if dS is not None and ctx.sink is not None:
            if ctx.sink.t is dS:
                dS = None  # accumulated into the sequence's shared gradient buffer (kernel epilogue)
                ctx.sink.release()
            else:
                dS = ctx.sink.deliver(dS)
        return dS, dQ, None, None, None, None


def _hsp_gemm_bwd(ctx, gs):
    """GEMM composition of the pooling VJP (fp32 parity path)."""
    S, Q, lengths, Pm, sc, lse, *outs = ctx.saved_tensors
    B, T, d = S.shape
    HQ = Q.shape[-2]
    G = Q.shape[0] if Q.dim() == 3 else 1
    dP = torch.empty(B, T, HQ, device=S.device, dtype=torch.float32)
    # D[b, c] = sum_t P dP = dO[c] . pooled[c]: the softmax-VJP column term
    # from the (B, HQ, d) pooled output instead of a pass over T
    Dcol = torch.empty(B, HQ, device=S.device, dtype=torch.float32)
    dS = None
    c0 = 0
    for g, n, o in zip(gs, ctx.splits, outs):
        g = torch.zeros(B, n, d, device=S.device, dtype=S.dtype) if g is None else g.contiguous()
        Dcol[:, c0:c0 + n] = torch.linalg.vecdot(g.float(), o.float())
        gemm(S, g.transpose(1, 2), dP[:, :, c0:c0 + n])
        if dS is None:
            dS = gemm(Pm[:, :, c0:c0 + n], g)
        else:
            gemm(Pm[:, :, c0:c0 + n], g, dS, beta=1.0)
        c0 += n
    dsc = torch.empty_like(Pm)
    lo = torch.empty_like(Pm) if Pm.dtype != torch.float32 else None
    a = _colsm_args(dsc, Pm, lengths)  # dtype_in = dsc dtype, dtype_out = P dtype
    a.X, a.x_rs, a.x_bs = sc.data_ptr(), sc.stride(1), sc.stride(0)  # recompute mode: P = exp(sc - LSE)
    a.LSE = lse.data_ptr()
    a.dP, a.dp_rs, a.dp_bs = dP.data_ptr(), dP.stride(1), dP.stride(0)
    a.dX, a.dx_rs, a.dx_bs = dsc.data_ptr(), dsc.stride(1), dsc.stride(0)
    a.dX_lo = lo.data_ptr() if lo is not None else None
    a.dtype_dp = _capi.dt(dP)
    a.Dcol = Dcol.data_ptr() if HSP_DCOL else None
    _capi.call("kl_colsoftmax_bwd", C.byref(a), _stream())
    Bg = B // G
    gemm(dsc.view(G, Bg, T, HQ), Q.view(G, 1, HQ, d).expand(G, Bg, HQ, d), dS.view(G, Bg, T, d), beta=1.0)
    # dQ = sum_b dsc^T S (over each query set's samples): softmax-VJP rows sum
    # to zero over t, so this reduction cancels; bf16 runs it on the hi + lo
    # split of dsc.
    dQ = torch.zeros(G, 1, HQ, d, device=S.device, dtype=torch.float32)
    gemm(dsc.view(G, Bg, T, HQ).transpose(2, 3), S.view(G, Bg, T, d), dQ, beta=1.0, reduce=(False, True))
    if lo is not None:
        gemm(lo.view(G, Bg, T, HQ).transpose(2, 3), S.view(G, Bg, T, d), dQ, beta=1.0, reduce=(False, True))
    dQ = dQ.reshape(Q.shape)
    return dS, dQ


HSP_FUSED = True  # tests flip this to A/B the fused tcgen05 pooling against the GEMM composition
HSP_BALANCED = True  # d = 512 forward: the balanced (split key range) kernel; False = one CTA per item


def _hsp_fused_ok(S, HQ, n_splits) -> bool:
    return (HSP_FUSED and S.dtype == torch.bfloat16 and S.shape[-1] in (128, 256, 512) and n_splits <= 2
            and bool(_capi.lib().kl_tcgen05_available()))


def _hsp_args(S, Q, lengths, n1, O1, O2, LSE):
    a = _capi.HspArgs()
    a.B, a.T, a.d = S.shape
    a.HQ, a.n1 = Q.shape[-2], n1
    a.q_group = a.B // Q.shape[0] if Q.dim() == 3 else 0
    a.dtype = _capi.dt(S)
    a.lengths = lengths.data_ptr()
    a.S, a.s_rs, a.s_bs = S.data_ptr(), S.stride(1), S.stride(0)
    a.Q = Q.data_ptr()
    a.O1, a.o1_bs = O1.data_ptr(), O1.stride(0)
    a.O2, a.o2_bs = O2.data_ptr(), O2.stride(0)
    a.LSE = LSE.data_ptr()
    return a


def _hsp_fused_bwd(ctx, gs):
    """kl_hsp_bwd: dS and the hi/lo score gradient dZ in one pass over S; then
    the batch-shared query gradient dQ = sum_b dZ S (hi + lo) as GEMMs."""
    S, Q, lengths, LSE, *outs = ctx.saved_tensors
    B, T, d = S.shape
    HQ = Q.shape[-2]
    G = Q.shape[0] if Q.dim() == 3 else 1
    # the pooled parts' gradients as one (B, HQ, d) row set (one kl_regroup;
    # missing gradients are zero rows); at d = 512 directly into the rows
    # [0, HQ) of the dS GEMM's K operand [dO; Qt] (B, 2 HQ, d)
    ns = [o.shape[1] for o in outs]
    wide = d == 512 and G == 1
    GQ = torch.empty(B, (2 if wide else 1) * HQ, d, device=S.device, dtype=S.dtype)
    segs, r0 = [], 0
    for g, n in zip(gs, ns):
        segs.append((None if g is None else (g if g.stride(2) == 1 else g.contiguous()), 0, GQ, r0, n))
        r0 += n
    if wide:
        segs.append((Q.unsqueeze(0).expand(B, HQ, d), 0, GQ, HQ, HQ))
    copy_rows(segs, B, d, S.dtype)
    dO = GQ[:, :HQ]
    # rowsum(dO * pooled) per part (the softmax-VJP term), no concatenated copy of the pooled rows
    Dq = torch.empty(B, HQ, device=S.device, dtype=torch.float32)
    r0 = 0
    for o, n in zip(outs, ns):
        _capi.call("kl_rowdot3", B, n, d, _capi.dt(o), dO[:, r0:].data_ptr(), dO.stride(0), dO.stride(1),
                   o.data_ptr(), o.stride(0), o.stride(1), Dq[:, r0:].data_ptr(), HQ, _stream())
        r0 += n
    acc = ctx.sink.take(S) if ctx.sink is not None else None
    if d == 512:
        return _hsp_bwd512(S, Q, lengths, LSE, dO, Dq, acc, ctx, GQ if wide else None)
    dS = acc if acc is not None else torch.empty_like(S)
    dZ = torch.empty(B, HQ, T, device=S.device, dtype=S.dtype)
    dZlo = torch.empty_like(dZ)
    a = _hsp_args(S, Q, lengths, HQ, dO, dO, LSE)
    a.dO1 = dO.data_ptr()
    a.dS, a.ds_rs, a.ds_bs = dS.data_ptr(), dS.stride(1), dS.stride(0)
    a.accumulate_ds = 1 if acc is not None else 0
    a.dZ, a.dZ_lo, a.Dq = dZ.data_ptr(), dZlo.data_ptr(), Dq.data_ptr()
    _capi.call("kl_hsp_bwd", C.byref(a), _stream())
    Bg = B // G
    dQ = zeros((G, 1, HQ, d), S.device)  # split-K partials add into it (fp32 reduce-add epilogue)
    gemm(dZ.view(G, Bg, HQ, T), S.view(G, Bg, T, d), dQ, beta=1.0, reduce=(False, True))
    gemm(dZlo.view(G, Bg, HQ, T), S.view(G, Bg, T, d), dQ, beta=1.0, reduce=(False, True))
    return dS, dQ.reshape(Q.shape)


def _hsp_bwd512(S, Q, lengths, LSE, dO, Dq, acc, ctx, GQ=None):
    """d = 512: kl_hsp_bwd writes P and dZ (one pass over S, the score
    products streamed through the kernel, hsp_bwd512_kernel) into PZ
    (B, 2 HQ, T) and dZ's bf16 residual into dZ_lo; the whole-width T-length
    products are tcgen05 GEMMs:
        dS  = [P; dZ]^T [dO; Qt]            (one GEMM, K = 2 HQ; accumulates
                                             into the shared sequence gradient)
        dQ  = sum_b (dZ + dZ_lo) S          (batch-reduced, hi + lo)."""
    B, T, d = S.shape
    HQ = Q.shape[-2]
    G = Q.shape[0] if Q.dim() == 3 else 1
    Bg = B // G
    PZ = torch.empty(B, 2 * HQ, T, device=S.device, dtype=S.dtype)
    dZlo = torch.empty(B, HQ, T, device=S.device, dtype=S.dtype)
    a = _hsp_args(S, Q, lengths, HQ, dO, dO, LSE)
    a.dO1 = dO.data_ptr()
    a.dS, a.ds_rs, a.ds_bs = S.data_ptr(), S.stride(1), S.stride(0)  # unused at d = 512
    a.dZ, a.dZ_lo, a.Dq = PZ.data_ptr(), dZlo.data_ptr(), Dq.data_ptr()
    _capi.call("kl_hsp_bwd", C.byref(a), _stream())
    if GQ is None:  # (grouped query sets: one per sample group)
        GQ = torch.cat([dO, Q.view(G, 1, HQ, d).expand(G, Bg, HQ, d).reshape(B, HQ, d)], dim=1)  # (B, 2 HQ, d)
    if acc is not None:
        dS = gemm(PZ.transpose(1, 2), GQ, acc, residual=acc)
    else:
        dS = gemm(PZ.transpose(1, 2), GQ)
    dQ = zeros((G, 1, HQ, d), S.device)
    gemm(PZ.view(G, Bg, 2 * HQ, T)[:, :, HQ:], S.view(G, Bg, T, d), dQ, beta=1.0, reduce=(False, True))
    gemm(dZlo.view(G, Bg, HQ, T), S.view(G, Bg, T, d), dQ, beta=1.0, reduce=(False, True))
    return dS, dQ.reshape(Q.shape)


# softmax-VJP column term of the composition path: False = the t-reduction
# sum_t P dP inside kl_colsoftmax_bwd, consistent with the fp32 P it
# recomputes (the bf16-rounded pooled output would put its rounding into the
# cancellation-heavy query gradient); True = rowdot(dO, pooled)
HSP_DCOL = False


def hsp_pool(S, Q, lengths, splits=None, n_recent=0, sink=None):
    """Pooled outputs, one (B, n, d) tensor per entry of ``splits`` (default:
    all HQ rows in one), then, if ``n_recent``, the recent rows (seqsum.py:
    186-196) — one op, so the sequence gets one gradient buffer.  ``Q`` is
    (HQ, d), or (G, HQ, d) for G grouped event types whose samples are
    stacked along S's batch (sample b pools with set b // (B / G))."""
    return _HspPool.apply(S, Q, lengths, tuple(splits) if splits else (Q.shape[-2],), int(n_recent), sink)


def _recent_fwd(S, lengths, n):
    B, T, d = S.shape
    if not S.is_contiguous():
        S = S.contiguous()
    out = torch.empty(B, n, d, device=S.device, dtype=S.dtype)
    _capi.call("kl_recent_rows_fwd", B, T, d, n, _capi.dt(S), S.data_ptr(), S.stride(0), lengths.data_ptr(),
               out.data_ptr(), out.stride(0), _stream())
    return out


def _recent_bwd_into(dS, g, lengths):
    """dS[b, len - n + r] += g[b, r] (kl_recent_rows_bwd accumulates)."""
    B, T, d = dS.shape
    g = g.contiguous()
    _capi.call("kl_recent_rows_bwd", B, T, d, g.shape[1], _capi.dt(g), g.data_ptr(), g.stride(0),
               lengths.data_ptr(), dS.data_ptr(), dS.stride(0), _stream())


# ---------------------------------------------------------------------------
def zeros(shape, device, dtype=torch.float32):
    """A zero-filled buffer as a memset (kl_memset: a memset node in the
    captured step, not an elementwise fill kernel)."""
    t = torch.empty(shape, device=device, dtype=dtype)
    if t.is_cuda:
        _capi.call("kl_memset", t.data_ptr(), t.numel() * t.element_size(), _stream())
    else:
        t.zero_()
    return t


def copy_rows(segs, B, d, dtype):
    """kl_regroup: segments (src tensor or None, src row, dst tensor, dst row,
    rows) over (B, n, d) row sets with unit column stride, all in one launch
    (chunks of MAX_SEGS segments)."""
    esz = 4 if dtype == torch.float32 else 2
    for c0 in range(0, len(segs), _capi.MAX_SEGS):
        chunk = [g for g in segs[c0:c0 + _capi.MAX_SEGS] if g[4] > 0]
        if not chunk:
            continue
        a = _capi.RegroupArgs()
        a.B, a.d, a.dtype, a.n_seg = B, d, _capi.dt(chunk[0][2]), len(chunk)
        for k, (src, r0, dst, q0, rows) in enumerate(chunk):
            g = a.seg[k]
            if src is not None:
                g.src = src.data_ptr() + r0 * src.stride(1) * esz
                g.src_bs, g.src_rs = src.stride(0), src.stride(1)
            g.dst = dst.data_ptr() + q0 * dst.stride(1) * esz
            g.dst_bs, g.dst_rs = dst.stride(0), dst.stride(1)
            g.rows = rows
        _capi.call("kl_regroup", C.byref(a), _stream())


def _plan(n_in, n_out):
    """Overlaps of two partitions of one token axis: (i, row in i, j, row in j, rows)."""
    out, i, j, ri, rj = [], 0, 0, 0, 0
    while i < len(n_in) and j < len(n_out):
        k = min(n_in[i] - ri, n_out[j] - rj)
        if k > 0:
            out.append((i, ri, j, rj, k))
        ri += k
        rj += k
        if ri == n_in[i]:
            i, ri = i + 1, 0
        if rj == n_out[j]:
            j, rj = j + 1, 0
    return out


class _Regroup(torch.autograd.Function):
    """Re-partition the token axis of (B, n_i, d) row sets into contiguous
    (B, m_j, d) tensors (sum n_i = sum m_j): torch.cat / slicing along dim 1
    without ATen copies, zero-fills or gradient accumulation — every row has
    exactly one source, so the VJP is the inverse regrouping (missing output
    gradients are zero rows).  One kl_regroup launch per direction."""

    @staticmethod
    def forward(ctx, sizes, *pieces):
        p0 = pieces[0]
        B, d = p0.shape[0], p0.shape[2]
        n_in = [t.shape[1] for t in pieces]
        outs = [torch.empty(B, m, d, device=p0.device, dtype=p0.dtype) for m in sizes]
        copy_rows([(pieces[i], ri, outs[j], rj, k) for i, ri, j, rj, k in _plan(n_in, sizes)], B, d, p0.dtype)
        ctx.n_in, ctx.sizes = n_in, tuple(sizes)
        return tuple(outs)

    @staticmethod
    def backward(ctx, *gs):
        ref = next(g for g in gs if g is not None)
        B, d = ref.shape[0], ref.shape[2]
        gin = [torch.empty(B, n, d, device=ref.device, dtype=ref.dtype) for n in ctx.n_in]
        gs = [g if g is None or g.stride(2) == 1 else g.contiguous() for g in gs]
        copy_rows([(gs[j], rj, gin[i], ri, k) for i, ri, j, rj, k in _plan(ctx.n_in, ctx.sizes)], B, d, ref.dtype)
        return (None,) + tuple(gin)


class _GatherRows(torch.autograd.Function):
    """Rows [a, b) of the token-axis concatenation of (B, n_i, d) pieces as one
    contiguous (B, b - a, d) tensor (one kl_regroup launch).  VJP: each
    touched piece's gradient in one launch — written whole where the range
    covers the piece, zero-filled (memset) around its rows otherwise."""

    @staticmethod
    def forward(ctx, a, b, *pieces):
        p0 = pieces[0]
        B, d = p0.shape[0], p0.shape[2]
        out = torch.empty(B, b - a, d, device=p0.device, dtype=p0.dtype)
        segs, lo = [], 0
        ctx.parts = []  # (piece index, row in piece, row in out, rows, covers the whole piece)
        for i, t in enumerate(pieces):
            n = t.shape[1]
            s0, s1 = max(a, lo), min(b, lo + n)
            if s0 < s1:
                segs.append((t if t.stride(2) == 1 else t.contiguous(), s0 - lo, out, s0 - a, s1 - s0))
                ctx.parts.append((i, s0 - lo, s0 - a, s1 - s0, s1 - s0 == n))
            lo += n
        copy_rows(segs, B, d, p0.dtype)
        ctx.shapes = [t.shape for t in pieces]
        return out

    @staticmethod
    def backward(ctx, g):
        g = g if g.stride(2) == 1 else g.contiguous()
        B, d = g.shape[0], g.shape[2]
        grads = [None] * len(ctx.shapes)
        segs = []
        for i, r_in, r_out, n, whole in ctx.parts:
            shape = tuple(ctx.shapes[i])
            gi = torch.empty(shape, device=g.device, dtype=g.dtype) if whole else zeros(shape, g.device, g.dtype)
            grads[i] = gi
            segs.append((g, r_out, gi, r_in, n))
        copy_rows(segs, B, d, g.dtype)
        return (None, None) + tuple(grads)


def gather_rows(pieces, a, b):
    """Rows [a, b) of torch.cat(pieces, dim=1) (see _GatherRows)."""
    if pieces[0].is_cuda:
        return _GatherRows.apply(int(a), int(b), *pieces)
    return torch.cat(pieces, dim=1)[:, a:b].contiguous()


def regroup(pieces, sizes):
    """(B, n_i, d) row sets -> contiguous (B, m_j, d) tensors over the same
    concatenated token axis (see _Regroup)."""
    if sum(t.shape[1] for t in pieces) != sum(sizes):
        raise ShapeError(f"regroup: {sum(t.shape[1] for t in pieces)} rows into {sum(sizes)}")
    return _Regroup.apply(tuple(int(m) for m in sizes), *pieces)


def cat_rows(pieces):
    """torch.cat(pieces, dim=1) of (B, n_i, d) row sets, one launch each way."""
    if len(pieces) == 1:
        return pieces[0]
    return regroup(pieces, [sum(t.shape[1] for t in pieces)])[0]


# ---------------------------------------------------------------------------
class _QueryFolds(torch.autograd.Function):
    """The batch-shared HSP seed / CLS query folds of several layers at once
    (seqsum.py:96-102, 26-34 with attention.py:85-89):
        seeds: Qt[l, q, h] = (RMSNorm(E_l) g_l)[q] W_q,l^h^T W_k,l^h * scale
        CLS:   Qt[l, q, h] = c_l[q] W_q,l'^h^T W_k,l'^h * scale
    as batched fp32 GEMMs over the layers (the per-layer parameter blocks are
    uniformly spaced in the flat buffer), rows ordered (query, head).  The
    backward runs once, after every layer's pooling backward, and writes the
    parameter gradients straight into the gradient buffer."""

    @staticmethod
    def forward(ctx, flat, P, keys, H, d_h, eps, stacked=False):
        seeds_k, gain_k, wqkv_k, cls_k, cw_k = keys
        E = P.stacked(seeds_k, "w32")
        G = P.stacked(gain_k, "w32")
        W = P.stacked(wqkv_k, "w32")
        L, n_s, d = E.shape
        Hd = H * d_h
        scale = 1.0 / float(d_h) ** 0.5
        xs = torch.empty(L, n_s, d, device=E.device, dtype=torch.float32)
        _capi.call("kl_rmsnorm_fwd_b", L, n_s, d, eps, E.data_ptr(), E.stride(0), G.data_ptr(), G.stride(0),
                   xs.data_ptr(), n_s * d, _stream())
        n_cls = P.shape(cls_k[0])[0] if cls_k else 0
        n_q = n_s + n_cls
        Q = torch.empty(L, n_q, H, d, device=E.device, dtype=torch.float32)
        qh_s = gemm(xs, W[:, :Hd].transpose(1, 2))  # (L, n_s, H*d_h)
        gemm(qh_s.view(L, n_s, H, d_h).permute(0, 2, 1, 3), W[:, Hd:2 * Hd].view(L, H, d_h, d),
             Q[:, :n_s].permute(0, 2, 1, 3), alpha=scale)
        qh_c = None
        if n_cls:
            Cq = P.stacked(cls_k, "w32")
            CW = P.stacked(cw_k, "w32")
            qh_c = gemm(Cq, CW[:, :Hd].transpose(1, 2))
            gemm(qh_c.view(L, n_cls, H, d_h).permute(0, 2, 1, 3), CW[:, Hd:2 * Hd].view(L, H, d_h, d),
                 Q[:, n_s:].permute(0, 2, 1, 3), alpha=scale)
        ctx.P, ctx.keys, ctx.H, ctx.d_h, ctx.eps = P, keys, H, d_h, eps
        ctx.save_for_backward(xs, qh_s, qh_c)
        Qr = Q.view(L, n_q * H, d)
        ctx.stacked = stacked
        return Qr if stacked else tuple(Qr[l] for l in range(L))

    @staticmethod
    def backward(ctx, *gs):
        P, (seeds_k, gain_k, wqkv_k, cls_k, cw_k) = ctx.P, ctx.keys
        xs, qh_s, qh_c = ctx.saved_tensors
        H, d_h = ctx.H, ctx.d_h
        L, n_s, d = xs.shape
        Hd = H * d_h
        scale = 1.0 / float(d_h) ** 0.5
        n_q = n_s + (P.shape(cls_k[0])[0] if cls_k else 0)
        if ctx.stacked:
            dQ = gs[0].contiguous().view(L, n_q, H, d)
        else:
            dQ = torch.stack([torch.zeros(n_q * H, d, device=xs.device) if g is None else g for g in gs])
            dQ = dQ.view(L, n_q, H, d)

        def fold_bwd(dQs, qh, n, W, gW):
            """dQs (L, H, n, d), qh (L, n, H*d_h): dW_k += scale qh^T dQ; returns
            dqh = scale dQ W_k^T as (L, n, H*d_h)."""
            dqh = torch.empty(L, n, H, d_h, device=xs.device, dtype=torch.float32)
            gemm(dQs, W[:, Hd:2 * Hd].view(L, H, d_h, d).transpose(2, 3), dqh.permute(0, 2, 1, 3), alpha=scale)
            gemm(qh.view(L, n, H, d_h).permute(0, 2, 3, 1), dQs, gW[:, Hd:2 * Hd].view(L, H, d_h, d),
                 alpha=scale, beta=1.0)
            return dqh.view(L, n, Hd)

        # seeds
        W = P.stacked(wqkv_k, "w32")
        gW = P.stacked(wqkv_k, "g")
        dq2 = fold_bwd(dQ[:, :n_s].permute(0, 2, 1, 3), qh_s, n_s, W, gW)
        gemm(dq2.transpose(1, 2), xs, gW[:, :Hd], beta=1.0)  # dW_q
        dxs = gemm(dq2, W[:, :Hd])  # (L, n_s, d)
        E = P.stacked(seeds_k, "w32")
        G = P.stacked(gain_k, "w32")
        gE = P.stacked(seeds_k, "g")
        gG = P.stacked(gain_k, "g")
        _capi.call("kl_rmsnorm_bwd_b", L, n_s, d, ctx.eps, E.data_ptr(), E.stride(0), G.data_ptr(), G.stride(0),
                   dxs.data_ptr(), n_s * d, gE.data_ptr(), gE.stride(0), gG.data_ptr(), gG.stride(0), 1, _stream())
        if cls_k:
            n_cls = P.shape(cls_k[0])[0]
            CW = P.stacked(cw_k, "w32")
            gCW = P.stacked(cw_k, "g")
            Cq = P.stacked(cls_k, "w32")
            dqc = fold_bwd(dQ[:, n_s:].permute(0, 2, 1, 3), qh_c, n_cls, CW, gCW)
            gemm(dqc.transpose(1, 2), Cq, gCW[:, :Hd], beta=1.0)
            gemm(dqc, CW[:, :Hd], P.stacked(cls_k, "g"), beta=1.0)
        return None, None, None, None, None, None, None


def query_folds(P, keys, H, d_h, eps=1e-6, stacked=False):
    """Per-entry (HQ, d) fp32 query rows of every entry in ``keys`` (lists of
    per-layer — or, for grouped event types, per-event — registry block
    keys), see _QueryFolds; one (n, HQ, d) tensor if ``stacked``; None if
    the blocks are not uniformly spaced."""
    for ks in keys:
        if ks and P.stacked(ks, "w32") is None:
            return None
    return _QueryFolds.apply(P.flat, P, keys, int(H), int(d_h), float(eps), bool(stacked))


# ---------------------------------------------------------------------------
class _RmsNorm(torch.autograd.Function):
    """rms_norm (tensor.py:552-556) on a batch-shared fp32 parameter block;
    dgain is written straight into the gradient buffer."""

    @staticmethod
    def forward(ctx, flat, P, xkey, gkey, eps):
        x = P.w32(xkey)
        gain = P.w32(gkey)
        rows, d = x.shape
        y = torch.empty(rows, d, device=x.device, dtype=torch.float32)
        _capi.call("kl_rmsnorm_fwd", rows, d, eps, x.data_ptr(), gain.data_ptr(), y.data_ptr(), _stream())
        ctx.P, ctx.xkey, ctx.gkey, ctx.eps = P, xkey, gkey, eps
        return y

    @staticmethod
    def backward(ctx, g):
        P = ctx.P
        x, gain = P.w32(ctx.xkey), P.w32(ctx.gkey)
        rows, d = x.shape
        g = g.contiguous().float()
        dx = torch.empty_like(g)
        dgain = torch.empty(d, device=g.device, dtype=torch.float32)
        _capi.call("kl_rmsnorm_bwd", rows, d, ctx.eps, x.data_ptr(), gain.data_ptr(), g.data_ptr(), dx.data_ptr(),
                   dgain.data_ptr(), _stream())
        P.g(ctx.xkey).add_(dx)
        P.g(ctx.gkey).add_(dgain)
        return None, None, None, None, None


def rms_norm_param(P, xkey, gkey, eps=1e-6):
    return _RmsNorm.apply(P.flat, P, xkey, gkey, float(eps))


class _Recent(torch.autograd.Function):
    """recent_rows (seqsum.py:186-196) on a padded batch."""

    @staticmethod
    def forward(ctx, S, lengths, n):
        B, T, d = S.shape
        out = torch.empty(B, n, d, device=S.device, dtype=S.dtype)
        _capi.call("kl_recent_rows_fwd", B, T, d, n, _capi.dt(S), S.data_ptr(), S.stride(0), lengths.data_ptr(),
                   out.data_ptr(), out.stride(0), _stream())
        ctx.save_for_backward(lengths)
        ctx.shape = S.shape
        return out

    @staticmethod
    def backward(ctx, g):
        (lengths,) = ctx.saved_tensors
        B, T, d = ctx.shape
        g = g.contiguous()
        dS = torch.zeros(B, T, d, device=g.device, dtype=g.dtype)
        _capi.call("kl_recent_rows_bwd", B, T, d, g.shape[1], _capi.dt(g), g.data_ptr(), g.stride(0),
                   lengths.data_ptr(), dS.data_ptr(), dS.stride(0), _stream())
        return dS, None, None


def recent_rows(S, lengths, n):
    if n == 0:
        return S.new_zeros(S.shape[0], 0, S.shape[2])
    if not S.is_contiguous():
        S = S.contiguous()
    return _Recent.apply(S, lengths, int(n))


def pad8(n: int) -> int:
    return (n + 7) // 8 * 8


class _GramTriu(torch.autograd.Function):
    """triu_flatten(x x^T) per sample (interaction.py:63-76, 116-117)."""

    @staticmethod
    def forward(ctx, x):
        B, n, d = x.shape
        if x.stride(2) != 1:
            raise ShapeError("gram_triu needs unit column stride")
        # pairs padded to a multiple of 8 (zeros) so the DotMap GEMM's rows are
        # 16-byte aligned for TMA; the padding multiplies zero weight columns
        tri = torch.empty(B, pad8(n * (n + 1) // 2), device=x.device, dtype=x.dtype)  # kernel zeroes the pad
        _capi.call("kl_gram_triu_fwd", B, n, d, _capi.dt(x), x.data_ptr(), x.stride(1), x.stride(0),
                   tri.data_ptr(), tri.stride(0), _stream())
        ctx.save_for_backward(x)
        return tri

    @staticmethod
    def backward(ctx, g):
        (x,) = ctx.saved_tensors
        B, n, d = x.shape
        g = g.contiguous()
        dx = torch.zeros(B, n, d, device=x.device, dtype=x.dtype)
        _capi.call("kl_gram_triu_bwd", B, n, d, _capi.dt(x), x.data_ptr(), x.stride(1), x.stride(0),
                   g.data_ptr(), g.stride(0), dx.data_ptr(), dx.stride(1), dx.stride(0), _stream())
        return dx


def gram_triu(x):
    return _GramTriu.apply(x)


class _Gated(torch.autograd.Function):
    """x + gate_deep*deep + gate_dot*dot (interaction.py:121); gates are
    (1,)-shaped fp32 parameters (interaction.py:97-98 with tensor.py:36)."""

    @staticmethod
    def forward(ctx, x, deep, dot, flat, P, gdkey, gtkey):
        B, n, d = deep.shape
        deep = deep.contiguous()
        dot = dot.contiguous()
        out = torch.empty(B, n, d, device=x.device, dtype=x.dtype)
        if x.stride(2) != 1 or x.stride(0) != n * x.stride(1):
            x = x.contiguous()
        _capi.call("kl_gated_sum_fwd", B * n, d, _capi.dt(x), x.data_ptr(), x.stride(1), deep.data_ptr(),
                   dot.data_ptr(), P.w32(gdkey).data_ptr(), P.w32(gtkey).data_ptr(), out.data_ptr(), d, _stream())
        ctx.save_for_backward(deep, dot)
        ctx.P, ctx.gdkey, ctx.gtkey = P, gdkey, gtkey
        return out

    @staticmethod
    def backward(ctx, g):
        deep, dot = ctx.saved_tensors
        P = ctx.P
        B, n, d = deep.shape
        g = g.contiguous()
        ddeep = torch.empty_like(deep)
        ddot = torch.empty_like(dot)
        scratch = torch.empty(2 * 512, device=g.device, dtype=torch.float64)
        dgd, dgt = P.g(ctx.gdkey), P.g(ctx.gtkey)  # fp32 (1,) views of the flat gradient: the kernel accumulates
        _capi.call("kl_gated_sum_bwd", B * n, d, _capi.dt(g), g.data_ptr(), d, deep.data_ptr(), dot.data_ptr(),
                   P.w32(ctx.gdkey).data_ptr(), P.w32(ctx.gtkey).data_ptr(), ddeep.data_ptr(), ddot.data_ptr(),
                   dgd.data_ptr(), dgt.data_ptr(), scratch.data_ptr(), _stream())
        return g, ddeep, ddot, None, None, None, None


def gated_sum(x, deep, dot, P, gdkey, gtkey):
    return _Gated.apply(x, deep, dot, P.flat, P, gdkey, gtkey)


class _WukongExpert(torch.autograd.Function):
    """One Wukong expert (interaction.py:106-121) as one autograd node:
        out = x + g_deep * (silu(x W1^T + b1) W2^T + b2) + g_dot * (triu(x x^T) W_dot^T)
    with the forward's kernels of gram_triu / the two linears / gated_sum.
    Its VJP accumulates the three input-gradient paths into one buffer — the
    deep path's dX GEMM takes the identity path (the incoming gradient) as its
    residual and the gram VJP adds in place — so autograd sees one consumer
    of x (no zero fills, clones or gradient additions between kernels)."""

    @staticmethod
    def forward(ctx, x, flat, P, dm, w1, b1, w2, b2, gd, gt):
        B, n, d = x.shape
        if x.stride(2) != 1 or x.stride(0) != n * x.stride(1) or x.stride(1) != d:
            x = x.contiguous()
        tri = torch.empty(B, pad8(n * (n + 1) // 2), device=x.device, dtype=x.dtype)  # kernel zeroes the pad
        _capi.call("kl_gram_triu_fwd", B, n, d, _capi.dt(x), x.data_ptr(), x.stride(1), x.stride(0),
                   tri.data_ptr(), tri.stride(0), _stream())
        dot = gemm(tri, P.w(dm).transpose(0, 1))  # (B, n*d)
        rows = x.view(B * n, d)
        H = P.w(w1).shape[0]
        pre = torch.empty(B * n, H, device=x.device, dtype=x.dtype)
        h1 = gemm(rows, P.w(w1).transpose(0, 1), bias=P.w32(b1), acts=_codes(["silu"]), aux=pre, aux_mode=1)
        deep = gemm(h1, P.w(w2).transpose(0, 1), bias=P.w32(b2))
        if numerics_check_mode() == "eager":
            flag_nonfinite(deep, "Mlp")
        out = torch.empty(B, n, d, device=x.device, dtype=x.dtype)
        _capi.call("kl_gated_sum_fwd", B * n, d, _capi.dt(x), x.data_ptr(), d, deep.data_ptr(), dot.data_ptr(),
                   P.w32(gd).data_ptr(), P.w32(gt).data_ptr(), out.data_ptr(), d, _stream())
        ctx.P, ctx.keys = P, (dm, w1, b1, w2, b2, gd, gt)
        ctx.save_for_backward(x, tri, pre, h1, deep, dot)
        return out

    @staticmethod
    def backward(ctx, g):
        x, tri, pre, h1, deep, dot = ctx.saved_tensors
        P = ctx.P
        dm, w1, b1, w2, b2, gd, gt = ctx.keys
        B, n, d = x.shape
        rows = B * n
        g = g.contiguous()
        ddeep = torch.empty_like(deep)
        ddot = torch.empty_like(dot)
        scratch = torch.empty(2 * 512, device=g.device, dtype=torch.float64)
        _capi.call("kl_gated_sum_bwd", rows, d, _capi.dt(g), g.data_ptr(), d, deep.data_ptr(), dot.data_ptr(),
                   P.w32(gd).data_ptr(), P.w32(gt).data_ptr(), ddeep.data_ptr(), ddot.data_ptr(),
                   P.g(gd).data_ptr(), P.g(gt).data_ptr(), scratch.data_ptr(), _stream())
        # deep path: dh1 = (ddeep W2) * silu'(pre); dx = dh1 W1 + g (the identity path)
        dh1 = gemm(ddeep, P.w(w2), acts=_codes(["silu"]), aux=pre, aux_mode=2)
        dx = gemm(dh1, P.w(w1), residual=g.view(rows, d))
        dtri = gemm(ddot, P.w(dm))  # dot path: d(triu) = ddot W_dot
        ones = _ones(rows, g.dtype, g.device)
        with _DwFork((ddeep, dh1, x, h1, ddot, tri, ones)):
            gemm(ddeep.t(), h1, P.g(w2), beta=1.0)
            gemm(ones.view(1, rows), ddeep, P.g(b2).view(1, -1), beta=1.0)
            gemm(dh1.t(), x.view(rows, d), P.g(w1), beta=1.0)
            gemm(ones.view(1, rows), dh1, P.g(b1).view(1, -1), beta=1.0)
            gemm(ddot.t(), tri, P.g(dm), beta=1.0)
        dx = dx.view(B, n, d)
        _capi.call("kl_gram_triu_bwd", B, n, d, _capi.dt(x), x.data_ptr(), x.stride(1), x.stride(0),
                   dtri.data_ptr(), dtri.stride(0), dx.data_ptr(), dx.stride(1), dx.stride(0), _stream())
        return dx, None, None, None, None, None, None, None, None, None


def wukong_expert_fused(x, P, dm, w1, b1, w2, b2, gd, gt):
    return _WukongExpert.apply(x, P.flat, P, dm, w1, b1, w2, b2, gd, gt)


class _BCE(torch.autograd.Function):
    """Mean BCE with logits (tensor.py:535-549), fp32."""

    @staticmethod
    def forward(ctx, z, y):
        z = z.contiguous().float()
        y = y.contiguous().float()
        loss = torch.empty(1, device=z.device, dtype=torch.float32)
        dz = torch.empty_like(z)
        _capi.call("kl_bce_fwd_bwd", z.numel(), z.data_ptr(), y.data_ptr(), loss.data_ptr(), dz.data_ptr(), _stream())
        ctx.save_for_backward(dz)
        return loss.view(())

    @staticmethod
    def backward(ctx, g):
        (dz,) = ctx.saved_tensors
        return dz * g, None


def bce_with_logits(z, y):
    return _BCE.apply(z, y)


class _Cast(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, dtype):
        ctx.src = x.dtype
        if x.dtype == dtype:
            return x
        x = x.contiguous()
        y = torch.empty(x.shape, device=x.device, dtype=dtype)
        _capi.call("kl_cast", x.numel(), _capi.dt(x), x.data_ptr(), _capi.dt(y), y.data_ptr(), _stream())
        return y

    @staticmethod
    def backward(ctx, g):
        if g.dtype == ctx.src:
            return g, None
        g = g.contiguous()
        y = torch.empty(g.shape, device=g.device, dtype=ctx.src)
        _capi.call("kl_cast", g.numel(), _capi.dt(g), g.data_ptr(), _capi.dt(y), y.data_ptr(), _stream())
        return y, None


def cast(x, dtype):
    return _Cast.apply(x, dtype)


class _HeadProj(torch.autograd.Function):
    """Per-head value projection + head concat of multi_head_attention
    (attention.py:88-92) on pooled rows laid out (B, n, H, d):
    out[b, i, h*d_h + c] = sum_f X[b,i,h,f] W_h[c,f].  One GEMM batched over
    the H heads with M = B*n rows (row stride H*d)."""

    @staticmethod
    def forward(ctx, X, flat, wref):
        B, n, H, d = X.shape
        W = wref.w()  # (H, d_h, d), or (G, H, d_h, d) for G grouped event types (samples stacked by group)
        G = W.shape[0] if W.dim() == 4 else 1
        W4 = W.view(G, *W.shape[-3:])
        d_h = W.shape[-2]
        X = X.contiguous()
        M = B // G * n
        out = torch.empty(B * n, H, d_h, device=X.device, dtype=X.dtype)
        gemm(X.view(G, M, H, d).permute(0, 2, 1, 3), W4.transpose(2, 3), out.view(G, M, H, d_h).permute(0, 2, 1, 3))
        ctx.save_for_backward(X)
        ctx.wref = wref
        return out.view(B, n, H * d_h)

    @staticmethod
    def backward(ctx, g):
        (X,) = ctx.saved_tensors
        B, n, H, d = X.shape
        W = ctx.wref.w()
        G = W.shape[0] if W.dim() == 4 else 1
        W4 = W.view(G, *W.shape[-3:])
        d_h = W.shape[-2]
        M = B // G * n
        gv = g.contiguous().view(G, M, H, d_h).permute(0, 2, 1, 3)  # (G, H, M, d_h)
        Xv = X.view(G, M, H, d).permute(0, 2, 1, 3)
        dX = torch.empty_like(X)
        gemm(gv, W4, dX.view(G, M, H, d).permute(0, 2, 1, 3))
        Wg = ctx.wref.g()
        gemm(gv.transpose(2, 3), Xv, Wg.view(G, *Wg.shape[-3:]), beta=1.0)
        return dX, None, None


def head_proj(X, wref):
    """X (B, n, H, d) -> (B, n, H*d_h)."""
    return _HeadProj.apply(X, wref.P.flat, wref)


class _RowsSelect(torch.autograd.Function):
    """out[b, t] = a[b, t] for t < lengths[b], else b_[b, t] (ablation paths:
    pass-through padding rows of an op without a residual)."""

    @staticmethod
    def forward(ctx, a, b_, lengths):
        T = a.shape[1]
        mask = (torch.arange(T, device=a.device)[None, :] < lengths[:, None].long())[..., None]
        ctx.save_for_backward(mask)
        return torch.where(mask, a, b_)

    @staticmethod
    def backward(ctx, g):
        (mask,) = ctx.saved_tensors
        z = torch.zeros((), device=g.device, dtype=g.dtype)
        return torch.where(mask, g, z), torch.where(mask, z, g), None


def rows_select(a, b_, lengths):
    return _RowsSelect.apply(a, b_, lengths)
