"""``kunlun.tensor`` — the reference module name (/root/reference/pkg/src/kunlun/tensor.py)
backed by the B200 implementation in ``paper_2602_10016_b200.tensor`` (same
names, dataclasses, validation and registry names; batched CUDA tensors)."""

from paper_2602_10016_b200.tensor import *  # noqa: F401,F403
