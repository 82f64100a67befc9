"""``kunlun.gdpa`` — the reference module name (/root/reference/pkg/src/kunlun/gdpa.py)
backed by the B200 implementation in ``paper_2602_10016_b200.gdpa`` (same
names, dataclasses, validation and registry names; batched CUDA tensors)."""

from paper_2602_10016_b200.gdpa import *  # noqa: F401,F403
