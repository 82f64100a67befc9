"""Adam over the flat parameter buffer (SPEC.md harness default:
beta1 .9, beta2 .999, eps 1e-8, lr 1e-3), one fused kernel that also
refreshes the bf16 compute mirror."""

from __future__ import annotations

import torch

from . import _capi


class FlatAdam:
    def __init__(self, P, lr=1e-3, betas=(0.9, 0.999), eps=1e-8):
        self.P = P
        self.lr, self.b1, self.b2, self.eps = lr, betas[0], betas[1], eps
        self.m = torch.zeros_like(P.gflat)
        self.v = torch.zeros_like(P.gflat)
        self.t = 0

    def step(self):
        self.t += 1
        P = self.P
        wc = P.flat_c.data_ptr() if P.flat_c is not None else None
        _capi.call("kl_adam_step", P.flat.numel(), self.lr, self.b1, self.b2, self.eps, self.t,
                   P.flat.data_ptr(), P.gflat.data_ptr(), self.m.data_ptr(), self.v.data_ptr(), wc, _capi._stream())
