"""CPU float64 oracle for the Kunlun layer hot path — TEST INFRASTRUCTURE ONLY.

This package restates, in plain numpy float64 with explicit hand-derived
vector-Jacobian products, the reference algorithm of arXiv 2602.10016's
``pkg/src/kunlun`` package (every function cites the reference file:line it
follows).  It is the *checker*: only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import it.
The product path (``paper_2602_10016_b200``) never imports it and fails
loudly when its CUDA library is missing.

Parity pinning: the restatement is pinned against golden vectors produced by
running the unmodified reference (``/root/reference/pkg/src/kunlun``) in the
build container — see ``tests/golden/make_golden.py`` and
``tests/test_oracle_golden.py``.  The reference ships no tests of its own
(SURVEY.md §4.1), so those fixtures plus the SPEC known-answer examples are
the pins.
"""

from .ops import ACT_CODES, act_fwd, act_dfn  # noqa: F401
