"""SPEC.md harness (lines 623-700): single-epoch trainer over the captured
training step, RunRecord stream, divergence checks, and the checkpoint
format's bitwise save -> load -> eval contract."""

import os

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _lib():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")


def _cfg():
    from paper_2602_10016_b200.model import EventConfig, ModelConfig

    return ModelConfig(L=2, d=64, heads=4, n_ctx=9, events=[EventConfig(T=64, w=16, budget=8, n_seeds=8, rank=2),
                                                          EventConfig(T=48, w=8, budget=4, n_seeds=4, rank=1)])


def test_train_records_and_checkpoint_roundtrip(tmp_path):
    from paper_2602_10016_b200.model import KunlunModel
    from paper_2602_10016_b200.optim import FlatAdam
    from paper_2602_10016_b200.trainer import (RunRecord, _device_batch, config_from_checkpoint, evaluate_ne,
                                               load_checkpoint, save_checkpoint, train)

    cfg = _cfg()
    model = KunlunModel(cfg, "cuda", torch.bfloat16, seed=1)
    opt = FlatAdam(model.P, lr=3e-3)
    recs = list(train(model, steps=30, batch=32, eval_every=10, opt=opt, seed=2))
    assert [r.step for r in recs] == [10, 20, 30]
    assert all(b.samples_seen > a.samples_seen for a, b in zip(recs, recs[1:]))
    assert all(np.isfinite([r.train_ne, r.eval_ne]).all() and r.gflops_per_sample > 0 for r in recs)
    assert recs[0].csv_row().count(",") == len(RunRecord.CSV_COLUMNS) - 1
    evset = [_device_batch(cfg, 32, 777, "cuda", torch.bfloat16)]
    ne0 = evaluate_ne(model, evset)
    path = os.path.join(tmp_path, "ck.npz")
    save_checkpoint(path, model, opt)
    cfg2 = config_from_checkpoint(path)
    assert cfg2 == cfg
    model2 = KunlunModel(cfg2, "cuda", torch.bfloat16, seed=99)
    opt2 = FlatAdam(model2.P)
    load_checkpoint(path, model2, opt2)
    assert torch.equal(model2.P.flat, model.P.flat) and torch.equal(opt2.m, opt.m) and torch.equal(opt2.t, opt.t)
    assert evaluate_ne(model2, evset) == ne0  # bitwise


def test_zero_lr_keeps_eval_ne():
    from paper_2602_10016_b200.model import KunlunModel
    from paper_2602_10016_b200.trainer import train

    model = KunlunModel(_cfg(), "cuda", torch.bfloat16, seed=1)
    recs = list(train(model, steps=20, batch=16, lr=0.0, eval_every=10, seed=3))
    assert recs[0].eval_ne == recs[1].eval_ne  # SPEC.md:649 "zero learning rate"
