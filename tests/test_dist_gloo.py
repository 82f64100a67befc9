"""Data-parallel gradient reduction (dist.GradReducer) on the CPU with the
gloo backend, world size 2: bucket ranges cover the flat gradient buffer,
per-layer buckets launched from the layer-boundary hooks in reverse order
(plus small-bucket merging) produce the exact average, and the sharded
batch's averaged gradient equals the full-batch gradient."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class _FakeCfg:
    def __init__(self, L):
        self.L = L


class _FakeModel:
    """Just enough of KunlunModel for the reducer: cfg.L, P (flat params with
    L{l}/pool blocks), layer_hook."""

    def __init__(self, L, sizes, late=()):
        from paper_2602_10016_b200.tensor import Params

        self._late = list(late)
        P = Params()
        for l in range(L):
            P.add(f"L{l}/pool", np.zeros((2, 3)))
            P.add(f"L{l}/w", np.zeros(sizes[l]))
        P.add("head/w0", np.zeros(5))
        P.finalize("cpu")
        self.P = P
        self.cfg = _FakeCfg(L)
        self.layer_hook = None

    def late_grad_blocks(self):
        return self._late


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, min_bucket, q, skip0=False, late=False):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2602_10016_b200.dist import GradReducer

    L = 4
    m = _FakeModel(L, [7, 1, 300, 2], late=["L2/w"] if late else [])
    red = GradReducer(m, min_bucket=min_bucket)
    # ranges tile [start of L0, end of buffer) without gaps
    assert red.ranges[0][0] == m.P.block_range("L0/pool")[0]
    for a, b in zip(red.ranges[:-1], red.ranges[1:]):
        assert a[1] == b[0]
    assert red.ranges[-1][1] == m.P.gflat.numel()
    g = torch.arange(m.P.gflat.numel(), dtype=torch.float32) * (rank + 1)
    m.P.gflat.copy_(g)
    for l in reversed(range(L)):  # backward order
        if skip0 and l == 0:
            continue  # layer 0's boundary never fires when its inputs need no gradient
        m.layer_hook(l)
    if late:  # a late contribution (like the query folds' backward) after every boundary
        lo, hi = m.P.block_range("L2/w")
        m.P.gflat[lo:hi] += 1000.0 * (rank + 1)
    red.finish()
    q.put((rank, m.P.gflat.numpy().copy()))
    dist.destroy_process_group()


@pytest.mark.parametrize("min_bucket,skip0,late", [(1, False, False), (64, False, False), (1, True, False),
                                                    (64, True, True), (1, False, True)])
def test_grad_average_world2(min_bucket, skip0, late):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, min_bucket, q, skip0, late)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = out[0].size
    expect = np.arange(n, dtype=np.float32) * 1.5  # mean of (1x, 2x)
    if late:
        from paper_2602_10016_b200.tensor import Params  # noqa: F401

        m = _FakeModel(4, [7, 1, 300, 2])
        lo, hi = m.P.block_range("L2/w")
        expect[lo:hi] += 1500.0
    start = 0
    for r in (0, 1):
        np.testing.assert_allclose(out[r][start:], expect[start:], rtol=0, atol=0)


def _shard_worker(rank, world, port, q):
    """Averaged per-rank gradients of a mean loss over a sharded batch equal
    the full-batch gradient (the DP invariant of SURVEY.md §8(e))."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    rng = np.random.default_rng(0)
    X = rng.normal(size=(8, 5))
    y = rng.normal(size=8)
    w = rng.normal(size=5)
    Xs, ys = X[rank * 4:(rank + 1) * 4], y[rank * 4:(rank + 1) * 4]
    g = torch.tensor(2 * Xs.T @ (Xs @ w - ys) / len(ys), dtype=torch.float64)
    dist.all_reduce(g)
    g /= world
    full = 2 * X.T @ (X @ w - y) / len(y)
    q.put(float(np.abs(g.numpy() - full).max()))
    dist.destroy_process_group()


def test_sharded_mean_gradient_equals_full_batch():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    errs = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert max(errs) < 1e-12
