"""Named workloads of BASELINE.json ``configs``, with the knobs the configs
leave open pinned from reference defaults:
n_kv=16 (gdpa.py:45), n_sum=4, tau=T, GDPA
activation cycle silu/relu/identity/tanh (gdpa.py:31), summary split
budget/4 : budget/2 : budget/4 (seqsum.py:141-145), expert hidden 2d, head
hidden 4d, M=2 experts."""

from __future__ import annotations

from .model import EventConfig, ModelConfig


def c1():
    """2-layer tiny: d=64, 4 heads, T=256, w=64, 8 HSP seeds, 4 event types, B=32."""
    ev = [EventConfig(T=256, w=64, budget=8, n_seeds=8, rank=2, name=f"ev{e}") for e in range(4)]
    return ModelConfig(L=2, d=64, heads=4, n_ctx=9, events=ev), 32


def c2():
    """4-layer d=256, T=1024, w=128 single-B200 BF16 with GDPA + HSP (1 event), B=128."""
    ev = [EventConfig(T=1024, w=128, budget=32, n_seeds=32, rank=8, name="click")]
    return ModelConfig(L=4, d=256, heads=4, n_ctx=16, events=ev), 128


def c3():
    """8-layer CompSkip, 16 event types (grouped over events), T=2048, B=32.
    Per-event budget 8 (2/4/2) and M=4 experts keep the Wukong DotMap
    (n_i*d x n_i(n_i+1)/2 per expert, interaction.py:90-91) at 6 M params;
    a 32-token budget x 16 events would make it 2.4 B params per expert."""
    ev = [EventConfig(T=2048, w=128, budget=8, n_seeds=8, rank=2, name=f"ev{e}") for e in range(16)]
    return ModelConfig(L=8, d=256, heads=4, n_ctx=16, events=ev, experts=4, compskip=True), 32


def c4():
    """8-layer d=512, 8 heads, T=4096, w=128, B=32 per GPU (weak scaling over 1/2/4/8)."""
    ev = [EventConfig(T=4096, w=128, budget=32, n_seeds=32, rank=8, name="click")]
    return ModelConfig(L=8, d=512, heads=8, n_ctx=16, events=ev), 32


CONFIGS = {"c1": c1, "c2": c2, "c3": c3, "c4": c4}
