"""``kunlun.model`` — the composed Kunlun layer / model (SPEC.md:451-533,
PAPER.md Alg. 1 and Alg. 4), which the reference package leaves to its SPEC;
backed by ``paper_2602_10016_b200.model``."""

from paper_2602_10016_b200.model import *  # noqa: F401,F403
