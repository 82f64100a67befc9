"""The reference-side adapter (paper_2602_10016_b200/refbind.py): reference
``Tensor``s through the C ABI, VJPs registered with ``record``
(tensor.py:185-195), against the float64 restatement at the FP32 tolerance."""

import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _tensor_module():
    """The real reference kunlun.tensor when importable (this container),
    else the contract restatement in tests/_reftape.py (GPU boxes)."""
    try:
        sys.path.insert(0, "/root/reference/pkg/src")
        import importlib

        mod = importlib.import_module("kunlun.tensor")
        if "reference" in (mod.__file__ or ""):
            return mod, True
    except Exception:
        pass
    finally:
        if sys.path and sys.path[0] == "/root/reference/pkg/src":
            sys.path.pop(0)
    from tests import _reftape

    return _reftape, False


@pytest.fixture(autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


@pytest.mark.parametrize("act", ["silu", "relu", "identity", "tanh", "sigmoid"])
def test_refbind_gdpa_core(act):
    from oracle.ops import act_dfn, act_fwd
    from paper_2602_10016_b200.refbind import bind
    from tests import _reftape

    T, real = _tensor_module()
    ops = bind(T)
    rng = np.random.default_rng(1)
    q, k, v = rng.normal(0, 1, (37, 16)), rng.normal(0, 1, (8, 16)), rng.normal(0, 1, (8, 16))
    g = rng.normal(0, 1, (37, 16))
    inv_tau = 1.0 / 3.0
    if real:  # the reference's own tape and backward
        qt, kt, vt = T.Tensor(q), T.Tensor(k), T.Tensor(v)
        for t in (qt, kt, vt):
            t.requires_grad = True
        with T.Tape() as tape:
            y = ops.gdpa_core(qt, kt, vt, act, inv_tau, 16, 4)
        node = tape.nodes[-1]
        dq, dk, dv = node.vjp(g)
    else:
        qt, kt, vt = (_reftape.Tensor(x, True) for x in (q, k, v))
        with _reftape.Tape() as tape:
            y = ops.gdpa_core(qt, kt, vt, act, inv_tau, 16, 4)
        grads = _reftape.backward(tape, y, g)
        dq, dk, dv = grads[id(qt)], grads[id(kt)], grads[id(vt)]
    assert y.requires_grad and len(tape.nodes) == 1
    z = (q @ k.T) * inv_tau
    a = act_fwd(act, z)
    ref = a @ v
    dz = (g @ v.T) * act_dfn(act, z, a) * inv_tau
    for got, want in ((y.data, ref), (dq, dz @ k), (dk, dz.T @ q), (dv, a.T @ g)):
        assert np.abs(got - want).max() <= 1e-5 * np.abs(want).max()


def test_refbind_matmul_and_errors():
    from paper_2602_10016_b200.refbind import bind
    from tests import _reftape

    ops = bind(_reftape)
    rng = np.random.default_rng(2)
    a, b = _reftape.Tensor(rng.normal(size=(9, 5)), True), _reftape.Tensor(rng.normal(size=(5, 7)), True)
    with _reftape.Tape() as tape:
        c = ops.matmul(a, b)
    g = rng.normal(size=(9, 7))
    grads = _reftape.backward(tape, c, g)
    assert np.abs(c.data - a.data @ b.data).max() < 1e-5 * np.abs(a.data @ b.data).max()
    assert np.abs(grads[id(a)] - g @ b.data.T).max() < 1e-5 * np.abs(g @ b.data.T).max()
    assert np.abs(grads[id(b)] - a.data.T @ g).max() < 1e-5 * np.abs(a.data.T @ g).max()
    with pytest.raises(ValueError):
        ops.gdpa_core(a, a, a, "nope", 1.0, 4, 4)
    with pytest.raises(ValueError):
        ops.gdpa_core(a, a, a, "silu", 1.0, 0, 4)
    big = _reftape.Tensor(np.full((4, 5), 60.0), True)
    with pytest.raises(_reftape.NumericsError):  # exp overflow -> _ensure_finite
        ops.gdpa_core(big, big, big, "exp", 1.0, 4, 4)
