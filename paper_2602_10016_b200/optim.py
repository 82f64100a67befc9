"""Adam over the flat parameter buffer (SPEC.md harness default:
beta1 .9, beta2 .999, eps 1e-8, lr 1e-3), one fused kernel that also
refreshes the bf16 compute mirror.  The step count lives on the device so a
captured training step (CUDA graph) replays correctly."""

from __future__ import annotations

import torch

from . import _capi


class FlatAdam:
    def __init__(self, P, lr=1e-3, betas=(0.9, 0.999), eps=1e-8):
        self.P = P
        self.lr, self.b1, self.b2, self.eps = lr, betas[0], betas[1], eps
        self.m = torch.zeros_like(P.gflat)
        self.v = torch.zeros_like(P.gflat)
        self.t = torch.zeros(1, dtype=torch.int32, device=P.gflat.device)

    def step(self):
        P = self.P
        wc = P.flat_c.data_ptr() if P.flat_c is not None else None
        _capi.call("kl_adam_step", P.flat.numel(), self.lr, self.b1, self.b2, self.eps, 0, self.t.data_ptr(),
                   P.flat.data_ptr(), P.gflat.data_ptr(), self.m.data_ptr(), self.v.data_ptr(), wc, _capi._stream())

    # one step split over parameter ranges: tick() once, then step_range()
    # over disjoint ranges covering the buffer (same arithmetic as step())
    def tick(self):
        _capi.call("kl_adam_tick", self.t.data_ptr(), _capi._stream())

    def step_range(self, lo: int, hi: int):
        P = self.P
        if hi <= lo:
            return
        e32, e16 = 4, 2
        wc = P.flat_c.data_ptr() + lo * e16 if P.flat_c is not None else None
        _capi.call("kl_adam_step", hi - lo, self.lr, self.b1, self.b2, self.eps, -1, self.t.data_ptr(),
                   P.flat.data_ptr() + lo * e32, P.gflat.data_ptr() + lo * e32, self.m.data_ptr() + lo * e32,
                   self.v.data_ptr() + lo * e32, wc, _capi._stream())


def _subtract(rng, holes, align: int = 1):
    """[lo, hi) minus the sorted disjoint ``holes``.  With ``align`` = 8 a
    hole's end is rounded up to the 8-element block alignment of Params (the
    gap is block padding, never a parameter), so every returned segment starts
    16-byte aligned as kl_adam_step requires, whatever the hole's size."""
    lo, hi = rng
    out = []
    for a, b in holes:
        b = min((b + align - 1) // align * align, hi) if b < hi else b
        if b <= lo or a >= hi:
            continue
        if a > lo:
            out.append((lo, a))
        lo = max(lo, b)
    if lo < hi:
        out.append((lo, hi))
    return out


class TrainStep:
    """One training step (zero grads, forward, BCE, backward, DP all-reduce,
    Adam) on static input buffers, optionally captured once as a CUDA graph
    and replayed: the step is ~400 kernel launches, whose host-side issue cost
    (ctypes + autograd) otherwise rivals the GPU time."""

    def __init__(self, model, opt, X, S, lengths, labels, reducer=None):
        self.model, self.opt, self.reducer = model, opt, reducer
        self.X, self.S, self.lengths, self.labels = X, S, lengths, labels
        self.graph = None
        self.loss = None
        # Adam split by layer (single process): a layer's parameters are
        # updated on a side stream as soon as its backward is done, beside the
        # earlier layers' backward; the query-fold inputs (gradients written
        # after layer 0) and the rest go last.  Data-parallel runs keep one
        # Adam after the all-reduce.
        self.segments = self.late = None
        if reducer is None and hasattr(model, "layer_param_ranges"):
            P = model.P
            holes = sorted(P.block_range(k) for k in model.late_grad_blocks())
            self.segments = [_subtract(r, holes, align=8) for r in model.layer_param_ranges()]
            covered = [seg for segs in self.segments for seg in segs]
            self.late = _subtract((0, P.gflat.numel()), sorted(covered))

    def _adam_layer(self, l):
        from . import functional as F

        self._fired.add(l)
        dev = self.X.device
        st = F.side_stream(dev, "adam")
        st.wait_stream(torch.cuda.current_stream(dev))
        for o in F.side_streams(dev):
            if o is not st:
                st.wait_stream(o)
        with torch.cuda.stream(st):
            for lo, hi in self.segments[l]:
                self.opt.step_range(lo, hi)

    def eager(self):
        from . import functional as F

        m = self.model
        split = F.BRANCH_STREAMS and self.segments is not None
        # the gradient buffer is cleared beside the forward (nothing writes it
        # before the backward, which waits for the clear)
        dev = self.X.device
        zs = None
        if self.X.is_cuda:
            zs = F.side_stream(dev, "zero_grad")
            zs.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(zs):
                m.P.zero_grad()
        else:
            m.P.zero_grad()
        if split:
            self.opt.tick()
            self._fired = set()
            m.layer_hook = self._adam_layer
        try:
            F.DW_STREAM_FWD = F.BRANCH_STREAMS
            loss, _ = m.loss(self.X, self.S, self.lengths, self.labels)
            F.DW_STREAM_FWD = False
            F.DW_STREAM = F.BRANCH_STREAMS  # weight-gradient GEMMs beside the dX chain
            if zs is not None:
                torch.cuda.current_stream(dev).wait_stream(zs)
            loss.backward()
        finally:
            F.DW_STREAM = F.DW_STREAM_FWD = False
            if split:
                m.layer_hook = None
        if F.BRANCH_STREAMS:  # (single-stream steps issued nothing on the side streams)
            F.dw_join(self.X.device)
        if self.reducer is not None:
            self.reducer.finish()
        if split:
            dev = self.X.device
            torch.cuda.current_stream(dev).wait_stream(F.side_stream(dev, "adam"))
            # layers whose boundary never fired (layer 0: its inputs are data
            # that need no gradient) and the late ranges
            for l in range(len(self.segments)):
                if l not in self._fired:
                    for lo, hi in self.segments[l]:
                        self.opt.step_range(lo, hi)
            for lo, hi in self.late:
                self.opt.step_range(lo, hi)
        else:
            self.opt.step()
        return loss

    def capture(self, warmup: int = 3):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            for _ in range(warmup):
                self.eager()
        torch.cuda.current_stream().wait_stream(s)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.loss = self.eager()
        self.graph = g
        return self

    def __call__(self):
        if self.graph is None:
            return self.eager()
        self.graph.replay()
        return self.loss

    def check_numerics(self):
        """NumericsError if any step since the last check produced a NaN / Inf
        logit or loss (the device flag of tensor.flag_nonfinite; one sync)."""
        from .tensor import raise_if_nonfinite

        raise_if_nonfinite(self.X.device, "training step")
