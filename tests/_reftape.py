"""Minimal restatement of the reference's tape contract for tests on boxes
without /root/reference (test infrastructure): ``Tensor`` holds ``data`` and
``requires_grad``; ``record(out, parents, vjp)`` sets ``out.requires_grad =
any(parent.requires_grad)`` and appends a node to the active tape
(tensor.py:185-195); ``backward`` sweeps the nodes in reverse
(tensor.py:198-230).  When the reference is importable the tests bind the
real ``kunlun.tensor`` instead."""

from __future__ import annotations

import numpy as np

_TAPES = []


class NumericsError(ArithmeticError):
    pass


class Tensor:
    def __init__(self, data, requires_grad=False):
        self.data = np.asarray(data, dtype=np.float64)
        self.requires_grad = requires_grad

    @property
    def shape(self):
        return self.data.shape


class Tape:
    def __init__(self):
        self.nodes = []

    def __enter__(self):
        _TAPES.append(self)
        return self

    def __exit__(self, *exc):
        _TAPES.pop()
        return False


def record(out, parents, vjp):
    out.requires_grad = any(p.requires_grad for p in parents)
    if _TAPES and out.requires_grad:
        _TAPES[-1].nodes.append((out, tuple(parents), vjp))
    return out


def backward(tape, out, seed):
    grads = {id(out): np.asarray(seed, dtype=np.float64)}
    for node_out, parents, vjp in reversed(tape.nodes):
        g = grads.get(id(node_out))
        if g is None:
            continue
        for p, gp in zip(parents, vjp(g)):
            if gp is not None and p.requires_grad:
                grads[id(p)] = grads.get(id(p), 0.0) + gp
    return grads
