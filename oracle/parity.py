"""Parity metrics (test infrastructure only).

Relative error of a tensor = max|got - ref| / max|ref| (norm-wise; an
elementwise ratio is meaningless near zeros).
Parameter gradients: in FP32 every tensor with more than one element is
held to its own scale (max-norm); scalar gradients (Wukong gates, the head's
output bias — sums with heavy cancellation) are held to the max of their
module's gradients.  In BF16 every gradient is compared in the Frobenius
norm against its module's gradient norm: ||got - ref||_2 / ||ref_module||_2.
(BF16 max-norm is ill-posed: a relu/threshold input within bf16 rounding of
its kink flips one derivative and moves a single element by O(1) relative,
a legitimate difference the 2-norm weighs by its share of the tensor.)
"""

from __future__ import annotations

import numpy as np

TOL_FP32 = 1e-5
TOL_BF16 = 2e-2


def rel(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if b.size == 0:
        return 0.0
    den = float(np.abs(b).max())
    num = float(np.abs(a - b).max())
    return num / den if den > 0 else num


def group(name: str) -> str:
    """Module of a registry name, without per-head / per-map indices."""
    parts = [q for q in name.split("/")[:-1]
             if not ((q.startswith("head") and q[4:].isdigit()) or (q.startswith("kron") and q[4:].isdigit()))]
    return "/".join(parts)


def grad_errors(got: dict, ref: dict, fp32: bool) -> dict:
    """name -> relative error under the rule in the module docstring."""
    scale: dict = {}
    for k, v in ref.items():
        g = group(k)
        if fp32:
            scale[g] = max(scale.get(g, 0.0), float(np.abs(v).max()) if v.size else 0.0)
        else:
            scale[g] = scale.get(g, 0.0) + float(np.sum(np.square(v, dtype=np.float64)))
    out = {}
    for k, v in ref.items():
        a = np.asarray(got[k], dtype=np.float64)
        if fp32:
            num = float(np.abs(a - v).max()) if v.size else 0.0
            den = float(np.abs(v).max()) if v.size > 1 else scale[group(k)]
        else:
            num = float(np.linalg.norm((a - v).ravel()))
            den = float(np.sqrt(scale[group(k)]))
        out[k] = num / den if den > 0 else num
    return out
