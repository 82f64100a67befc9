"""Reference-side binding of the C ABI: the B200 kernels as fused ops of the
reference numpy package, registered through its plugin hook
``record(out, parents, vjp)`` (/root/reference/pkg/src/kunlun/tensor.py:185-195).

This is what a maintainer of the reference would add to route its matmul and
its in-tree fused op ``gdpa_core`` (gdpa.py:141-187) through
libkunlun_sm100a.so: reference ``Tensor``s in, reference
``Tensor``s out, the VJP recorded on the reference's tape.  Device buffers
are torch CUDA tensors (plumbing); every product is a ``kl_gemm`` call on the
FP32 path (the 1e-5 parity path), with the activation and its derivative in
the GEMM epilogue (aux_mode 1 saves Z, aux_mode 2 applies Act'(Z)).

    from kunlun import tensor as T          # the reference package
    ops = bind(T)
    y = ops.gdpa_core(q, k, v, "silu", 1 / tau, 64, 16)   # recorded on T's tape
"""

from __future__ import annotations

import numpy as np
import torch

from . import _capi
from .tensor import ACTIVATIONS, NumericsError


class RefBinding:
    """Fused ops for a reference tensor module (needs ``Tensor`` and ``record``)."""

    def __init__(self, tensor_module, device: str = "cuda"):
        self.T = tensor_module
        self.device = device
        self._numerics = getattr(tensor_module, "NumericsError", NumericsError)

    # -- plumbing ---------------------------------------------------------
    def _dev(self, x) -> torch.Tensor:
        return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float32), device=self.device)

    def _host(self, t: torch.Tensor) -> np.ndarray:
        out = t.double().cpu().numpy()
        if not np.isfinite(out).all():  # _ensure_finite (tensor.py:21-27)
            raise self._numerics("non-finite values from a B200 fused op")
        return out

    def _wrap(self, data):
        return self.T.Tensor(data)

    # -- ops ----------------------------------------------------------------
    def matmul(self, a, b):
        """tensor.matmul (tensor.py:283-289): C = A B; VJP dA = g B^T, dB = A^T g."""
        A, B = self._dev(a.data), self._dev(b.data)
        out = self._wrap(self._host(_capi.gemm(A, B)))

        def vjp(g):
            G = self._dev(g)
            return self._host(_capi.gemm(G, B.t())), self._host(_capi.gemm(A.t(), G))

        return self.T.record(out, (a, b), vjp)

    def gdpa_core(self, q, k, v, act: str, inv_tau: float, block_t: int = 128, block_kv: int = 16):
        """gdpa.py:141-187: Act(Q K^T * inv_tau) V and its VJP
        dZ = (g V^T) * Act'(Z) * inv_tau, dQ = dZ K, dK = dZ^T Q, dV = Act(Z)^T g.
        The device contraction is untiled (block_t / block_kv only shape the
        reference's Python loop; validated as there)."""
        if block_t < 1 or block_kv < 1:
            raise ValueError("tile sizes must be >= 1")
        if act not in ACTIVATIONS:
            raise ValueError(f"unknown activation {act!r}")
        Q, K, V = self._dev(q.data), self._dev(k.data), self._dev(v.data)
        T_, n_kv = Q.shape[0], K.shape[0]
        Z = torch.empty(T_, n_kv, device=self.device)
        A = _capi.gemm(Q, K.t(), alpha=float(inv_tau), acts=[act], aux=Z, aux_mode=1)  # A = Act(Z), Z saved
        out = self._wrap(self._host(_capi.gemm(A, V)))

        def vjp(g):
            G = self._dev(g)
            dZ = torch.empty_like(Z)
            _capi.gemm(G, V.t(), dZ, alpha=float(inv_tau), acts=[act], aux=Z, aux_mode=2)
            return (self._host(_capi.gemm(dZ, K)), self._host(_capi.gemm(dZ.t(), Q)),
                    self._host(_capi.gemm(A.t(), G)))

        return self.T.record(out, (q, k, v), vjp)


def bind(tensor_module, device: str = "cuda") -> RefBinding:
    return RefBinding(tensor_module, device)
