"""Operator-API vocabulary shared with the reference numcore
(/root/reference/pkg/src/kunlun/tensor.py): the error types, the activation
tags, and the named parameter registry.

On the B200 path a "tensor" is a ``torch.Tensor`` on the GPU (batched
``(B, T, d)`` plus ``lengths``), and the reference's ``record(out, parents,
vjp)`` plugin hook (tensor.py:185-195) is played by the
``torch.autograd.Function`` wrappers in ``functional.py`` that call the
CUDA library through the C ABI.
"""

from __future__ import annotations

import math

import numpy as np
import torch


class ShapeError(ValueError):
    """Operand shapes do not satisfy an op's contract (tensor.py:17-18)."""


class NumericsError(ArithmeticError):
    """An op produced NaN/Inf, or training diverged (tensor.py:21-22)."""


# Tag -> C-ABI code, reference table order (tensor.py:431-440).
ACTIVATIONS = {"identity": 0, "relu": 1, "silu": 2, "tanh": 3, "sigmoid": 4, "exp": 5, "sqrt": 6, "log": 7}


def _sel(view: torch.Tensor, index):
    """A registry name's view of its block: an index expression, or a
    callable (e.g. a transposed slice) for blocks packed in a kernel layout."""
    return index(view) if callable(index) else view[index]


class Params:
    """Ordered registry of named learnable tensors (tensor.py:105-144),
    stored in one flat fp32 device buffer.

    * ``block(key, shape)`` reserves a packed block (e.g. all heads' Q/K/V
      projections stacked as one (3*H*d_h, d) matrix) and returns ``key``;
      ``add(name, data, block=key, index=...)`` registers a reference
      registry name as a view into it.  ``add(name, data)`` alone reserves a
      block of the name's own shape.
    * ``finalize(device, compute_dtype)`` allocates ``flat`` (fp32 master
      values), ``gflat`` (fp32 gradients, written by the kernels'
      weight-gradient epilogues), and — for bf16 compute — ``flat_c``, the
      bf16 mirror refreshed once per step by one cast kernel.
    * ``w(key)`` is the compute-dtype view the kernels read, ``g(key)`` the
      fp32 gradient view the backward kernels accumulate into.

    One flat gradient buffer is also what the data-parallel reducer
    all-reduces in buckets (dist.py).
    """

    def __init__(self):
        self._blocks: dict[str, tuple[int, tuple]] = {}
        self._names: dict[str, tuple[str, object]] = {}
        self._pending: list[tuple[str, object, object]] = []
        self._size = 0
        self.flat = None
        self.gflat = None
        self.flat_c = None
        self.device = None
        self.compute_dtype = torch.float32

    # -- layout ------------------------------------------------------------
    def block(self, key: str, shape) -> str:
        if key in self._blocks:
            raise ValueError(f"duplicate parameter block {key!r}")
        shape = tuple(int(s) for s in shape)
        n = int(np.prod(shape)) if shape else 1
        # 16-byte alignment of every block (TMA / vector loads, bf16 and fp32)
        off = (self._size + 7) // 8 * 8
        self._blocks[key] = (off, shape)
        self._size = off + n
        return key

    def add(self, name: str, data=None, *, block: str | None = None, index=()) -> str:
        if name in self._names:
            raise ValueError(f"duplicate parameter name {name!r}")
        if block is None:
            block = self.block(name, np.shape(data))
            index = ()
        self._names[name] = (block, index)
        if data is not None:
            self._pending.append((block, index, np.asarray(data, dtype=np.float32)))
        return name

    def finalize(self, device, compute_dtype=torch.float32) -> "Params":
        self.device = torch.device(device)
        self.compute_dtype = compute_dtype
        n = max(1, (self._size + 63) // 64 * 64)
        self.flat = torch.zeros(n, dtype=torch.float32, device=self.device)
        self.flat.requires_grad_(True)
        self.gflat = torch.zeros(n, dtype=torch.float32, device=self.device)
        if compute_dtype != torch.float32:
            self.flat_c = torch.empty(n, dtype=compute_dtype, device=self.device)
        with torch.no_grad():
            for block, index, arr in self._pending:
                _sel(self._view(self.flat.detach(), block), index).copy_(torch.from_numpy(arr))
        self._pending = []
        self.refresh()
        return self

    def _view(self, buf, key):
        off, shape = self._blocks[key]
        n = int(np.prod(shape)) if shape else 1
        return buf[off: off + n].view(shape)

    # -- access --------------------------------------------------------------
    def w(self, key: str) -> torch.Tensor:
        """Compute-dtype view of a block (no autograd; see functional.py)."""
        buf = self.flat_c if self.flat_c is not None else self.flat.detach()
        return self._view(buf, key)

    def w32(self, key: str) -> torch.Tensor:
        return self._view(self.flat.detach(), key)

    def g(self, key: str) -> torch.Tensor:
        return self._view(self.gflat, key)

    def shape(self, key: str):
        return self._blocks[key][1]

    def refresh(self) -> None:
        """Re-cast the fp32 masters into the compute-dtype mirror (one kernel)."""
        if self.flat_c is not None:
            from . import _capi
            _capi.call("kl_cast", self.flat.numel(), _capi.KL_F32, self.flat.data_ptr(), _capi.KL_BF16,
                       self.flat_c.data_ptr(), _capi._stream())

    def stacked(self, keys, which: str = "w"):
        """(len(keys),) + shape view over equally-shaped blocks whose offsets
        are uniformly spaced in the flat buffers (e.g. one block per layer:
        every layer creates its parameters in the same order), so a batched
        GEMM can address all of them; ``which`` = "w" (compute dtype), "w32"
        or "g".  None if the blocks are not uniformly spaced."""
        offs = [self._blocks[k][0] for k in keys]
        shape = self._blocks[keys[0]][1]
        if any(self._blocks[k][1] != shape for k in keys):
            return None
        st = offs[1] - offs[0] if len(offs) > 1 else int(np.prod(shape)) if shape else 1
        if st <= 0 or any(offs[i + 1] - offs[i] != st for i in range(len(offs) - 1)):
            return None
        base = {"w": self.flat_c if self.flat_c is not None else self.flat.detach(), "w32": self.flat.detach(),
                "g": self.gflat}[which]
        inner = []
        acc = 1
        for dim in reversed(shape):
            inner.insert(0, acc)
            acc *= dim
        return base.as_strided((len(keys),) + tuple(shape), (st,) + tuple(inner), offs[0])

    def zero_grad(self) -> None:
        if self.gflat.is_cuda:  # a memset (node), not an elementwise fill kernel
            from . import _capi

            _capi.call("kl_memset", self.gflat.data_ptr(), self.gflat.numel() * 4,
                       torch.cuda.current_stream(self.gflat.device).cuda_stream)
        else:
            self.gflat.zero_()

    # -- reference-registry views --------------------------------------------
    def __getitem__(self, name: str) -> torch.Tensor:
        block, index = self._names[name]
        return _sel(self.w32(block), index)

    def __contains__(self, name: str) -> bool:
        return name in self._names

    def __len__(self) -> int:
        return len(self._names)

    def names(self) -> list[str]:
        return list(self._names)

    def items(self):
        return [(n, self[n]) for n in self._names]

    def count(self) -> int:
        """Total learnable scalars."""
        return sum(int(np.prod(self[n].shape)) for n in self._names)

    def grad(self, name: str) -> torch.Tensor:
        block, index = self._names[name]
        return _sel(self.g(block), index)

    def set(self, name: str, data) -> None:
        """Replace a parameter's value (trainer-only, between steps)."""
        arr = torch.as_tensor(np.asarray(data), dtype=torch.float32)
        cur = self[name]
        if tuple(arr.shape) != tuple(cur.shape):
            raise ShapeError(f"parameter {name!r} has shape {tuple(cur.shape)}, got {tuple(arr.shape)}")
        if not torch.isfinite(arr).all():
            raise NumericsError(f"non-finite values in parameter update of {name!r}")
        with torch.no_grad():
            cur.copy_(arr.to(cur.device))

    def load(self, named: dict) -> None:
        for k, v in named.items():
            if k in self._names:
                self.set(k, v)
        self.refresh()

    def block_of(self, name: str):
        return self._names[name]

    def block_range(self, key: str) -> tuple[int, int]:
        off, shape = self._blocks[key]
        return off, off + (int(np.prod(shape)) if shape else 1)

    @staticmethod
    def normal(rng, std, shape):
        return rng.normal(0.0, std, shape)


def inv_sqrt(x: float) -> float:
    return 1.0 / math.sqrt(x)


# ---------------------------------------------------------------------------
# Non-finite detection (the reference's _ensure_finite, tensor.py:21-27,
# called from every op at tensor.py:245-549).
#
# The device path cannot raise inside a kernel, so a scan kernel
# (kl_check_finite) ORs a per-device flag and the host raises NumericsError
# when it reads it.  Modes (set_numerics_check):
#   "eager"     every public op (gdpa_forward, mha_window / mha_full,
#               multi_head_attention, hsp_summarize, pma, global_interaction,
#               Mlp, the model's logits / loss) scans its output and raises
#               at once — the reference's semantics, one host sync per op;
#   "deferred"  (default) only the model's logits and loss are scanned (a NaN
#               / Inf anywhere upstream reaches them), with no sync; the flag
#               is read by raise_if_nonfinite() — TrainStep.check_numerics()
#               and bench.py call it once after the steps;
#   "off"       no scans.
_NUMERICS = {"mode": "deferred"}
_FLAGS: dict = {}


def set_numerics_check(mode: str) -> None:
    if mode not in ("eager", "deferred", "off"):
        raise ValueError(f"numerics check mode must be eager, deferred or off, got {mode!r}")
    _NUMERICS["mode"] = mode


def numerics_check_mode() -> str:
    return _NUMERICS["mode"]


def _flag(device) -> torch.Tensor:
    key = torch.device(device).index or 0
    f = _FLAGS.get(key)
    if f is None:
        f = torch.zeros(1, dtype=torch.int32, device=device)
        _FLAGS[key] = f
    return f


def flag_nonfinite(t: torch.Tensor, what: str = "") -> None:
    """Scan ``t`` on its stream and OR the device's non-finite flag; in
    eager mode raise NumericsError now if it is set."""
    mode = _NUMERICS["mode"]
    if mode == "off" or t is None or not t.is_cuda or t.numel() == 0:
        return
    from . import _capi

    x = t.detach()
    if not x.is_contiguous():
        x = x.contiguous()
    f = _flag(x.device)
    _capi.call("kl_check_finite", x.numel(), _capi.dt(x), x.data_ptr(), f.data_ptr(), _capi._stream())
    if mode == "eager":
        raise_if_nonfinite(x.device, what)


def raise_if_nonfinite(device="cuda", what: str = "") -> None:
    """Read (and clear) the device's non-finite flag; NumericsError if set."""
    f = _flag(device)
    if int(f.item()):
        f.zero_()
        raise NumericsError(f"non-finite values{' in ' + what if what else ''} (NaN/Inf; tensor.py:21-27)")
