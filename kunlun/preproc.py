"""``kunlun.preproc`` — the reference module name (/root/reference/pkg/src/kunlun/preproc.py)
backed by the B200 implementation in ``paper_2602_10016_b200.preproc`` (same
names, dataclasses, validation and registry names; batched CUDA tensors)."""

from paper_2602_10016_b200.preproc import *  # noqa: F401,F403
