"""Data parallelism with the real model: two
ranks on one GPU (gloo process group on CUDA tensors — host-side copies, no
kernels that wait on each other), each running KunlunModel on its half of a
global batch with the per-layer GradReducer buckets launched from the
backward's layer-boundary hooks; after GradReducer.finish() every rank's
averaged gradient equals the single-process full-batch gradient.

(The NCCL path differs only in the process-group backend and runs inside
the captured training step in bench.py; a gloo all-reduce cannot be
captured in a CUDA graph, so this test runs the eager step.)"""

import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _setup():
    from paper_2602_10016_b200.model import EventConfig, ModelConfig
    from paper_2602_10016_b200.synth import ctr_batch

    cfg = ModelConfig(L=3, d=256, heads=4, n_ctx=16, events=[EventConfig(T=384, w=128, budget=8, n_seeds=8, rank=2)])
    Xn, Sn, Ln, yn = ctr_batch(cfg, 4, seed=11)
    Ln = [np.array([384, 200, 1, 384], dtype=np.int32)]
    return cfg, Xn, Sn, Ln, yn


def _grads(model, X, S, lens, y, reducer=None):
    model.P.zero_grad()
    loss, _ = model.loss(X, S, lens, y)
    loss.backward()
    if reducer is not None:
        reducer.finish()
    torch.cuda.synchronize()
    return model.P.gflat.detach().double().cpu().numpy()


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2602_10016_b200.dist import GradReducer
        from paper_2602_10016_b200.model import KunlunModel

        cfg, Xn, Sn, Ln, yn = _setup()
        dev = torch.device("cuda", 0)
        bf = torch.bfloat16
        model = KunlunModel(cfg, dev, bf, seed=0)
        full = None
        if rank == 0:  # the single-process full-batch reference gradient
            full = _grads(model, torch.tensor(Xn, device=dev).to(bf), [torch.tensor(s, device=dev).to(bf) for s in Sn],
                          [torch.tensor(l, device=dev) for l in Ln], torch.tensor(yn, device=dev))
        red = GradReducer(model, min_bucket=1 << 16)
        sl = slice(2 * rank, 2 * rank + 2)
        g = _grads(model, torch.tensor(Xn[sl], device=dev).to(bf), [torch.tensor(s[sl], device=dev).to(bf) for s in Sn],
                   [torch.tensor(l[sl], device=dev) for l in Ln], torch.tensor(yn[sl], device=dev), red)
        out = {"g": g}
        if rank == 0:
            errs = {}
            for name in model.P.names():
                key, _ = model.P.block_of(name)
                lo, hi = model.P.block_range(key)
                a, b = g[lo:hi], full[lo:hi]
                den = np.linalg.norm(b)
                errs[key] = float(np.linalg.norm(a - b) / den) if den > 0 else float(np.abs(a).max())
            out["errs"] = errs
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_dp_two_ranks_real_model_matches_full_batch():
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=600) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # both ranks hold the same averaged gradient
    assert np.array_equal(res[0]["g"], res[1]["g"])
    errs = res[0]["errs"]
    worst = sorted(errs.items(), key=lambda kv: -kv[1])[:5]
    assert all(e < 1e-2 for e in errs.values()), worst
