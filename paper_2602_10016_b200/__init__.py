"""B200-native Kunlun layer hot path (arXiv 2602.10016).

Drop-in for the reference package's operator API (``kunlun.gdpa``,
``kunlun.attention``, ``kunlun.seqsum``, ``kunlun.interaction``,
``kunlun.mlp``, ``kunlun.jagged``, ``kunlun.tensor``) plus the SPEC-only
``model`` / ``metrics`` pieces, over batched CUDA tensors.  Every device op
runs hand-written sm_100a kernels from ``lib/libkunlun_sm100a.so`` through
the C ABI in ``include/kunlun_capi.h``; there is no CPU fallback.
"""

from . import tensor  # noqa: F401
from .tensor import ACTIVATIONS, NumericsError, Params, ShapeError  # noqa: F401

__all__ = ["tensor", "ACTIVATIONS", "NumericsError", "Params", "ShapeError"]


def load_library():
    """Load libkunlun_sm100a.so (raises if it has not been built)."""
    from . import _capi

    return _capi.lib()
