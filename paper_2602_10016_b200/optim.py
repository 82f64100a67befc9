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

    def eager(self):
        from . import functional as F

        m = self.model
        m.P.zero_grad()
        loss, _ = m.loss(self.X, self.S, self.lengths, self.labels)
        F.DW_STREAM = F.BRANCH_STREAMS  # weight-gradient GEMMs beside the dX chain
        try:
            loss.backward()
        finally:
            F.DW_STREAM = False
        F.dw_join(self.X.device)
        if self.reducer is not None:
            self.reducer.finish()
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
