"""Single-epoch trainer and checkpoint format (SPEC.md harness module,
lines 623-700), over the captured B200 training step.

* ``train`` streams synthetic CTR batches (synth.ctr_batch; SPEC's
  SyntheticSpec reduced to what the layer path consumes) through one CUDA-graph
  captured ``TrainStep`` (forward, BCE, backward, fused Adam — the SPEC's
  Adam-style default β1 .9, β2 .999, ε 1e-8, lr 1e-3), evaluates NE (kl_ne)
  on a held-out interleaved slice every ``eval_every`` steps and yields one
  ``RunRecord`` per interval (step, samples_seen, train_ne,
  eval_ne, gflops_per_sample, qps, wall_time_s).  Divergence (NE > 10 or a
  non-finite loss) aborts with NumericsError.
* Checkpoints are one ``.npz``: the registry-named fp32 parameters, the Adam
  moments and step, and the model config as JSON — ``load_checkpoint``
  restores them bit for bit, so save -> load -> eval reproduces the eval NE
  exactly.
"""

from __future__ import annotations

import dataclasses
import json
import time
from dataclasses import dataclass

import numpy as np
import torch

from . import functional as F
from . import metrics
from .model import EventConfig, KunlunModel, ModelConfig
from .optim import FlatAdam, TrainStep
from .synth import ctr_batch
from .tensor import NumericsError


@dataclass
class RunRecord:
    step: int
    samples_seen: int
    train_ne: float
    eval_ne: float
    gflops_per_sample: float
    qps: float
    wall_time_s: float

    CSV_COLUMNS = ("step", "samples_seen", "train_ne", "eval_ne", "gflops_per_sample", "qps", "wall_time_s")

    def csv_row(self) -> str:
        return ",".join(str(getattr(self, c)) for c in self.CSV_COLUMNS)


def _device_batch(cfg, B, seed, device, dtype):
    Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=seed, full_length=False)
    return (torch.tensor(Xn, device=device).to(dtype), [torch.tensor(s, device=device).to(dtype) for s in Sn],
            [torch.tensor(l, device=device) for l in Ln], torch.tensor(yn, device=device))


def evaluate_ne(model: KunlunModel, batches) -> float:
    """NE of the model's logits over ``batches`` (no grad)."""
    zs, ys = [], []
    with torch.no_grad():
        for X, S, L, y in batches:
            zs.append(model.forward(X, S, L).float())
            ys.append(y.float())
    return metrics.normalized_entropy(torch.cat(ys), torch.cat(zs), from_logits=True).ne


def train(model: KunlunModel, steps: int, batch: int, *, lr: float = 1e-3, seed: int = 0, eval_every: int = 10,
          eval_batches: int = 2, graph: bool = True, opt: FlatAdam | None = None):
    """Single-pass streaming training; yields a RunRecord every
    ``eval_every`` steps (and after the last).  Batch i of the stream uses
    seed ``seed * 1_000_003 + i``; the eval slice is every 10th batch index
    (held out, "eval slice 10% of the stream, interleaved")."""
    cfg = model.cfg
    dev, dt = model.P.device, model.dtype
    opt = opt or FlatAdam(model.P, lr=lr)
    train_ids = [i for i in range(steps + steps // 9 + 2) if i % 10 != 9][:steps]
    eval_ids = [i for i in range(10 * eval_batches) if i % 10 == 9][:eval_batches]
    eval_set = [_device_batch(cfg, batch, seed * 1_000_003 + i, dev, dt) for i in eval_ids]
    X, S, L, y = _device_batch(cfg, batch, seed * 1_000_003 + train_ids[0], dev, dt)
    if model.groups is not None:  # grouped event types read the sequences as one stacked batch
        from .grouped import stage

        S, L = stage(S), stage(L)
    step = TrainStep(model, opt, X, S, L, y)
    if graph:
        step.eager()  # warm-up before capture (also the first training update)
        step.capture(warmup=0)
        done = 1
    else:
        done = 0
    flops = metrics.train_flops_per_sample(cfg, model.flags, model.seq_live())
    t0 = time.perf_counter()
    seen, zs, ys = batch * done, [], []
    for k in range(done, steps):
        Xn, Sn, Ln, yn = _device_batch(cfg, batch, seed * 1_000_003 + train_ids[k], dev, dt)
        step.X.copy_(Xn)
        for a, b in zip(step.S, Sn):
            a.copy_(b)
        for a, b in zip(step.lengths, Ln):
            a.copy_(b)
        step.labels.copy_(yn)
        loss = step()
        seen += batch
        if (k + 1) % eval_every == 0 or k + 1 == steps:
            torch.cuda.synchronize()
            lv = float(loss.detach())
            if not np.isfinite(lv):
                raise NumericsError(f"training diverged at step {k + 1}: loss {lv}")
            step.check_numerics()
            wall = time.perf_counter() - t0
            ev = evaluate_ne(model, eval_set)
            tr = evaluate_ne(model, [(step.X, step.S, step.lengths, step.labels)])
            if ev > 10 or not np.isfinite(ev):
                raise NumericsError(f"training diverged at step {k + 1}: eval NE {ev}")
            yield RunRecord(k + 1, seen, tr, ev, flops / 1e9, seen / max(wall, 1e-9), wall)


# ---------------------------------------------------------------------------
# checkpoints


def save_checkpoint(path: str, model: KunlunModel, opt: FlatAdam | None = None) -> None:
    """One .npz: ``param:<registry name>`` fp32 arrays, ``adam:m`` / ``adam:v``
    (flat fp32) and ``adam:t``, ``config`` (ModelConfig as JSON) and
    ``format`` = "kunlun-b200-ckpt-v1"."""
    P = model.P
    torch.cuda.synchronize()
    arrays = {f"param:{n}": P[n].detach().cpu().numpy() for n in P.names()}
    arrays["flat"] = P.flat.detach().cpu().numpy()
    if opt is not None:
        arrays["adam:m"] = opt.m.cpu().numpy()
        arrays["adam:v"] = opt.v.cpu().numpy()
        arrays["adam:t"] = opt.t.cpu().numpy()
        arrays["adam:hyper"] = np.array([opt.lr, opt.b1, opt.b2, opt.eps])
    cfg = dataclasses.asdict(model.cfg)
    arrays["config"] = np.array(json.dumps(cfg))
    arrays["format"] = np.array("kunlun-b200-ckpt-v1")
    np.savez(path, **arrays)


def config_from_checkpoint(path: str) -> ModelConfig:
    z = np.load(path, allow_pickle=False)
    cfg = json.loads(str(z["config"]))
    cfg["events"] = [EventConfig(**e) for e in cfg["events"]]
    cfg["gdpa_acts"] = tuple(cfg["gdpa_acts"])
    return ModelConfig(**cfg)


def load_checkpoint(path: str, model: KunlunModel, opt: FlatAdam | None = None) -> None:
    """Restore parameters (the flat fp32 master buffer, bit for bit, then the
    compute mirror) and, if given, the Adam state."""
    z = np.load(path, allow_pickle=False)
    if str(z["format"]) != "kunlun-b200-ckpt-v1":
        raise ValueError(f"not a kunlun-b200 checkpoint: {path}")
    P = model.P
    flat = torch.from_numpy(z["flat"])
    if flat.numel() != P.flat.numel():
        raise ValueError("checkpoint parameter layout does not match the model")
    with torch.no_grad():
        P.flat.copy_(flat.to(P.flat.device))
    P.refresh()
    if opt is not None and "adam:m" in z.files:
        opt.m.copy_(torch.from_numpy(z["adam:m"]).to(opt.m.device))
        opt.v.copy_(torch.from_numpy(z["adam:v"]).to(opt.v.device))
        opt.t.copy_(torch.from_numpy(z["adam:t"]).to(opt.t.device))
