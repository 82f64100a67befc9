"""Data-parallel gradient reduction (NCCL over NVLink 5 / NVSwitch).

The path shards by batch: every rank runs the full model
on its slice of samples; the only exchange is the average of the fp32
parameter gradients.  Gradients already live in ONE flat buffer
(``Params.gflat``) laid out in parameter-creation order, so each layer's
parameters form one contiguous bucket.  The model's per-layer boundary hook
fires when autograd has finished that layer's backward; the reducer then
records an event on the compute stream and launches the layer's all-reduce
on a dedicated communication stream, overlapping the remaining backward.
``finish()`` makes the compute stream wait for all buckets (before the
optimizer).  Buckets smaller than ``min_bucket`` elements are merged with
the next one to amortise launch latency.
"""

from __future__ import annotations

import torch
import torch.distributed as dist

from . import functional as F


class GradReducer:
    def __init__(self, model, group=None, min_bucket: int = 1 << 20, average: bool = True):
        self.model = model
        self.P = model.P
        self.group = group
        self.world = dist.get_world_size(group)
        self.average = average
        self.min_bucket = min_bucket
        L = model.cfg.L
        # element ranges of each layer's parameters (+ the head with the last layer)
        bounds = [self._layer_start(l) for l in range(L)] + [self.P.gflat.numel()]
        self.ranges = [(bounds[l], bounds[l + 1]) for l in range(L)]
        # blocks whose gradients are written after every layer's backward
        # (the query-fold inputs, model.late_grad_blocks) are reduced in
        # finish(), not with their layer's bucket
        from .optim import _subtract

        holes = sorted(self.P.block_range(k) for k in model.late_grad_blocks()) \
            if hasattr(model, "late_grad_blocks") else []
        self.segments = [_subtract(r, holes) for r in self.ranges]
        self.late = holes
        self.stream = torch.cuda.Stream() if self.P.gflat.is_cuda else None
        self.pending = []
        self._carry = None
        self._done = set()
        model.layer_hook = self.on_layer_done

    def _layer_start(self, l: int) -> int:
        key, _ = self.P.block_of(f"L{l}/pool")
        return self.P.block_range(key)[0]

    def _launch(self, lo: int, hi: int):
        buf = self.P.gflat[lo:hi]
        if self.stream is not None:
            ev = torch.cuda.Event()
            ev.record()
            with torch.cuda.stream(self.stream):
                self.stream.wait_event(ev)
                # the layer's gradients are also written on the parallel
                # branch and weight-gradient streams (functional.run_branches,
                # DW_STREAM): everything they were given so far precedes this
                for st in F.side_streams(buf.device):
                    self.stream.wait_stream(st)
                dist.all_reduce(buf, group=self.group)
                if self.average:
                    buf.mul_(1.0 / self.world)
        else:
            dist.all_reduce(buf, group=self.group)
            if self.average:
                buf.mul_(1.0 / self.world)

    def on_layer_done(self, l: int):
        self._done.add(l)
        segs = (self._carry or []) + self.segments[l]
        self._carry = None
        if sum(b - a for a, b in segs) < self.min_bucket and l > 0:
            self._carry = segs
            return
        for lo, hi in segs:
            self._launch(lo, hi)

    def finish(self):
        segs = self._carry or []
        self._carry = None
        # layers whose boundary never fired (layer 0 when its inputs are data
        # that need no gradient), then the late blocks
        for l in range(len(self.ranges)):
            if l not in self._done:
                segs += self.segments[l]
        segs += self.late
        for lo, hi in segs:
            self._launch(lo, hi)
        self._done = set()
        if self.stream is not None:
            torch.cuda.current_stream().wait_stream(self.stream)
