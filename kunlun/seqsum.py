"""``kunlun.seqsum`` — the reference module name (/root/reference/pkg/src/kunlun/seqsum.py)
backed by the B200 implementation in ``paper_2602_10016_b200.seqsum`` (same
names, dataclasses, validation and registry names; batched CUDA tensors)."""

from paper_2602_10016_b200.seqsum import *  # noqa: F401,F403
