"""Parity metrics (test infrastructure only).

Every tensor is held to its OWN scale (BASELINE.json north_star: FP32 within
1e-5 relative, BF16 within 2e-2 relative, per output / logit / gradient):

* FP32: max-norm relative error  max|got - ref| / max|ref|.
* BF16: Frobenius relative error ||got - ref||_2 / ||ref||_2.  (An elementwise
  max ratio is ill-posed in bf16: an input within bf16 rounding of a relu /
  threshold kink flips one derivative and moves that single element by O(1)
  relative — a legitimate difference the 2-norm weighs by its share of the
  tensor.)

Documented exception 1 — the relu kink (bf16 only): the fused GDPA kernels
compute Z = S Kt^T from the bf16-stored fold Kt = K W_q (the device's
operand format), whose rounding (2^-9 relative) flips the sign of Z for the
~0.1% of entries that sit within rounding of 0; each flip switches relu'
between 0 and 1 for that entry.  The derivative is discontinuous there, so
the gradients that sum dZ over the sequence — dKt = dZ^T S, hence the relu
heads' w_q and w_kgen gradients, and the non-sequence pooling matrix whose
gradient sums every head's dK — move by ~2-7% in the Frobenius norm while
everything else stays at bf16 rounding.  Those tensors (``relu_kink``) are
held to KINK_TOL = 1e-1 against this oracle AND, in
tests/test_gpu_parity.py::test_gdpa_vs_oracle, to the 2e-2 bf16 tolerance
against the same oracle evaluated with the device's own relu mask (Z from the
device's bf16 Kt), which isolates the kink from any kernel error.

Documented exception 2: a gradient with ONE element (the (1,)-shaped
Wukong gates, interaction.py:97-98 with tensor.py:36, and the head's output
bias) is a sum over the whole batch with heavy cancellation, so its own
magnitude can be arbitrarily small; it is held to the norm of its module's
gradients instead (max-norm in FP32, 2-norm in BF16).  A tensor whose
reference is exactly zero is compared in absolute terms.
"""

from __future__ import annotations

import numpy as np

TOL_FP32 = 1e-5
TOL_BF16 = 2e-2
KINK_TOL = 1e-1


def rel(a, b) -> float:
    """Max-norm relative error (the FP32 rule)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if b.size == 0:
        return 0.0
    den = float(np.abs(b).max())
    num = float(np.abs(a - b).max())
    return num / den if den > 0 else num


def relf(a, b) -> float:
    """Frobenius relative error (the BF16 rule)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if b.size == 0:
        return 0.0
    den = float(np.linalg.norm(b.ravel()))
    num = float(np.linalg.norm((a - b).ravel()))
    return num / den if den > 0 else num


def err(a, b, fp32: bool) -> float:
    return rel(a, b) if fp32 else relf(a, b)


def group(name: str) -> str:
    """Module of a registry name, without per-head / per-map indices."""
    parts = [q for q in name.split("/")[:-1]
             if not ((q.startswith("head") and q[4:].isdigit()) or (q.startswith("kron") and q[4:].isdigit()))]
    return "/".join(parts)


def grad_errors(got: dict, ref: dict, fp32: bool) -> dict:
    """name -> relative error under the per-tensor rule in the module
    docstring (one-element tensors: against their module's scale)."""
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
        v = np.asarray(v, dtype=np.float64)
        if v.size > 1:
            out[k] = err(a, v, fp32)
            continue
        num = float(np.abs(a - v).max()) if v.size else 0.0
        den = scale[group(k)] if fp32 else float(np.sqrt(scale[group(k)]))
        out[k] = num / den if den > 0 else num
    return out


def relu_kink(names, acts_of, pools=()) -> set:
    """Gradient names that exception 1 covers: ``{p}/head{h}/w_q`` and
    ``{p}/head{h}/w_kgen`` of GDPA blocks whose head h uses relu, plus the
    names in ``pools`` (the non-sequence pooling matrices P whose gradient
    sums every head's dK: dP = dX_sum X^T, dX_sum = sum_h KG_h^T vec(dK_h)).
    ``acts_of(prefix)`` returns that block's activation tags, or None if the
    prefix is not a GDPA block."""
    out = set(n for n in names if n in set(pools))
    for n in names:
        parts = n.split("/")
        if len(parts) < 3 or parts[-1] not in ("w_q", "w_kgen") or not parts[-2].startswith("head"):
            continue
        prefix = "/".join(parts[:-2])
        acts = acts_of(prefix)
        h = int(parts[-2][4:])
        if acts and acts[h % len(acts)] == "relu":
            out.add(n)
    return out


def violations(errs: dict, fp32: bool, kink=()) -> list:
    """(name, err, tol) of every tensor over its tolerance."""
    out = []
    for k, e in errs.items():
        tol = TOL_FP32 if fp32 else (KINK_TOL if k in kink else TOL_BF16)
        if not e < tol:
            out.append((k, e, tol))
    return sorted(out, key=lambda x: -x[1])
