"""Drop-in import name for the Kunlun hot path on B200.

``import kunlun.gdpa`` / ``kunlun.attention`` / ``kunlun.seqsum`` /
``kunlun.interaction`` / ``kunlun.mlp`` / ``kunlun.jagged`` / ``kunlun.tensor``
/ ``kunlun.preproc`` resolve to the B200 modules of ``paper_2602_10016_b200``,
which keep the reference package's (/root/reference/pkg/src/kunlun) function
names, dataclasses, validation messages and parameter registry names, over
batched ``(B, T, d)`` CUDA tensors with per-sample ``lengths``.  ``kunlun.model``
adds the composed layer (SPEC layer_forward / CompSkip) the reference leaves to
its SPEC.  There is no CPU fallback: the ops raise if the sm_100a library or
the GPU is missing.
"""

from paper_2602_10016_b200 import load_library  # noqa: F401
from paper_2602_10016_b200.tensor import ACTIVATIONS, NumericsError, ShapeError  # noqa: F401

from . import attention, gdpa, interaction, jagged, mlp, preproc, seqsum, tensor  # noqa: F401,E402
