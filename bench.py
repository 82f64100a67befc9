#!/usr/bin/env python
"""Kunlun fwd+bwd training-step throughput on B200 (BASELINE.json metric:
samples/sec and MFU vs B200 BF16 peak at 1/2/4/8 GPUs).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl b200|reference]

N > 1 is launched by torchrun (one process per GPU, NCCL).  A step = zero
grads + forward of all layers + BCE + backward + DP gradient all-reduce +
fused Adam, on a synthetic CTR batch of the named config.  Rank 0 prints one
JSON line.  ``--impl reference`` times the reference CPU algorithm (the
float64 oracle restatement, oracle/) on the host cores instead.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return p["bf16_tflops"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), p["hbm_gbs"], "measured"
    except Exception:
        return 1590.0, 1400.0, 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
            except ValueError:
                continue
            for n, v in zip(names, r[2:]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU reference (oracle restatement of the reference algorithm) — checker only


def _cpu_worker(args):
    spec_name, n, seed = args
    import numpy as np

    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from oracle import model as OM

    spec, p = _CPU_STATE[spec_name]
    rng = np.random.default_rng(seed)
    X = rng.normal(0, 1 / np.sqrt(spec.d), (n, spec.n_ctx, spec.d))
    S = [rng.normal(0, 1 / np.sqrt(spec.d), (n, ev.T, spec.d)) for ev in spec.events]
    lengths = [np.full(n, ev.T) for ev in spec.events]
    labels = (rng.random(n) < 0.2).astype(np.float64)
    OM.model_forward_backward(spec, p, X, S, lengths, labels)
    return n


_CPU_STATE = {}


def oracle_spec(cfg):
    from oracle import model as OM

    return OM.ModelSpec(L=cfg.L, d=cfg.d, heads=cfg.heads, n_ctx=cfg.n_ctx, n_sum=cfg.n_sum, n_kv=cfg.n_kv,
                        experts=cfg.experts, compskip=cfg.compskip, gdpa_acts=tuple(cfg.gdpa_acts),
                        expert_hidden=cfg.expert_hidden, head_hidden=cfg.head_hidden,
                        events=[OM.EventSpec(T=e.T, w=e.w, budget=e.budget, n_seeds=e.n_seeds, rank=e.rank,
                                             causal=e.causal) for e in cfg.events])


def cpu_reference(cfg, workers: int, samples_per_worker: int = 1, rounds: int = 1, warm: int = 0):
    """Times the float64 oracle fwd+bwd (the reference algorithm restated,
    oracle/model.py) with ``workers`` forked single-thread processes, each on
    ``samples_per_worker`` samples per round.  Returns per-round samples/s."""
    import multiprocessing as mp

    from oracle import model as OM

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    spec = oracle_spec(cfg)
    _CPU_STATE["spec"] = (spec, OM.init_params(spec, seed=0))
    ctx = mp.get_context("fork")
    rates = []
    with ctx.Pool(workers) as pool:
        for r in range(warm + rounds):
            t0 = time.perf_counter()
            done = sum(pool.map(_cpu_worker, [("spec", samples_per_worker, 1000 * r + i) for i in range(workers)]))
            dt = time.perf_counter() - t0
            if r >= warm:
                rates.append(done / dt)
    return rates


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------


def run_reference(args, cfg, B, rank, world):
    """--impl reference: the reference CPU algorithm on this box's host cores."""
    if rank != 0:
        return
    workers = max(1, min(host_cores(), args.cpu_workers))
    rates = cpu_reference(cfg, workers, 1, rounds=args.steps, warm=args.warmup)
    v = statistics.median(rates)
    line = {
        "impl": "reference", "metric": "kunlun_fwd_bwd_samples_per_s", "value": v, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * workers / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload(args, cfg, B, world),
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": workers, "kind": "port",
                         "sample": f"{workers} samples/step (1 per worker process), oracle float64 fwd+bwd"},
        "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def graph_census(log, step, use_graph):
    """Per-call-site device time of one (graph-replayed) training step:
    CUPTI kernel records (torch.profiler) of the step, matched in launch order
    to the C-ABI calls of an eager step (``log``: entry, shape, site, isolated
    ms, kernels launched).  Printed to stderr."""
    import collections

    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    kern = sorted([e for e in prof.events() if e.device_type.name == "CUDA"], key=lambda e: e.time_range.start)
    ours = [e for e in kern if e.name.startswith(("kl::", "void kl::", "gdpa::", "void gdpa::"))]
    other = [e for e in kern if e not in ours]
    step_us = (kern[-1].time_range.end - kern[0].time_range.start) if kern else 0.0
    sites = []
    for name, shape, site, _, nl in log:
        sites += [(name, shape, site)] * nl
    by_fn, by_site, cnt = collections.defaultdict(float), collections.defaultdict(float), collections.Counter()
    for i, e in enumerate(ours):
        nm, shape, site = sites[i] if i < len(sites) else ("?", "", "?")
        dur = e.time_range.end - e.time_range.start
        by_fn[(nm, site.split("<")[0])] += dur
        by_site[(nm, shape, site)] += dur
        cnt[(nm, shape, site)] += 1
    kt = collections.defaultdict(float)
    for e in kern:
        kt[e.name[:90]] += e.time_range.end - e.time_range.start
    tot = sum(kt.values())
    print(f"graph census ({'graph' if use_graph else 'eager'} step): {len(kern)} kernels, {len(ours)} ours "
          f"({len(sites)} expected), kernel time {tot / 1e3:.3f} ms, first->last {step_us / 1e3:.3f} ms; "
          f"torch-native kernels {sum(e.time_range.end - e.time_range.start for e in other) / 1e3:.3f} ms",
          file=sys.stderr)
    durs = sorted(e.time_range.end - e.time_range.start for e in kern)
    for lo_, hi_ in ((0, 5), (5, 10), (10, 20), (20, 50), (50, 1e9)):
        sel = [x for x in durs if lo_ <= x < hi_]
        print(f"  kernels {lo_:>3}-{hi_:<4} us: {len(sel):4d}, {sum(sel) / 1e3:7.3f} ms", file=sys.stderr)
    print("--- by kernel", file=sys.stderr)
    for k, v in sorted(kt.items(), key=lambda kv: -kv[1])[:30]:
        print(f"{v / 1e3:8.3f} ms {100 * v / tot:5.1f}%  {k}", file=sys.stderr)
    print("--- by call site", file=sys.stderr)
    for k, v in sorted(by_site.items(), key=lambda kv: -kv[1])[:150]:
        print(f"{v / 1e3:8.3f} ms {100 * v / tot:5.1f}% {cnt[k]:4d}k  {k[0]:18s} {k[1]:24s} {k[2]}", file=sys.stderr)


def workload(args, cfg, B, world):
    ev = cfg.events[0]
    return {"workload": f"kunlun_{args.config}_train_step", "model": "kunlun", "layers": cfg.L, "d": cfg.d,
            "heads": cfg.heads, "seq_len": ev.T, "window": ev.w, "events": len(cfg.events),
            "n_seeds": ev.n_seeds, "budget": ev.budget, "kron_rank": ev.rank, "n_ctx": cfg.n_ctx,
            "n_kv": cfg.n_kv, "n_sum": cfg.n_sum, "experts": cfg.experts, "compskip": cfg.compskip,
            "batch_per_gpu": B, "global_batch": B * world, "parallelism": f"dp{world}",
            "l2": "per-step working set (activations, several GB) >> 126 MB L2"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-workers", type=int, default=32)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gemm-census", action="store_true", help="log every kl_gemm shape/path of one step to stderr")
    ap.add_argument("--op-census", action="store_true",
                    help="time every C-ABI call of one eager step in isolation, grouped by call site (stderr)")
    ap.add_argument("--eager", action="store_true", help="issue every kernel from Python each step (no CUDA graph)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2602_10016_b200.configs import CONFIGS

    cfg, B = CONFIGS[args.config]()
    if args.batch:
        B = args.batch

    if args.impl == "reference":
        run_reference(args, cfg, B, rank, world)
        return

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2602_10016_b200 import _capi, metrics
    from paper_2602_10016_b200 import functional as F
    from paper_2602_10016_b200.model import KunlunModel
    from paper_2602_10016_b200.optim import FlatAdam
    from paper_2602_10016_b200.synth import ctr_batch

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    _capi.lib()
    dtype = torch.bfloat16
    model = KunlunModel(cfg, dev, dtype, seed=0)
    opt = FlatAdam(model.P)
    reducer = None
    if world > 1:
        from paper_2602_10016_b200.dist import GradReducer

        reducer = GradReducer(model)

    Xn, Sn, Ln, yn = ctr_batch(cfg, B, seed=1234 + rank)
    X = torch.tensor(Xn, device=dev).to(dtype)
    S = [torch.tensor(s, device=dev).to(dtype) for s in Sn]
    lens = [torch.tensor(l, device=dev) for l in Ln]
    y = torch.tensor(yn, device=dev)

    from paper_2602_10016_b200.optim import TrainStep

    bufs = [(X, S, y)]
    if not args.no_e2e:  # a second static input set: the e2e loop double-buffers host->device copies
        bufs.append((torch.empty_like(X), [torch.empty_like(s) for s in S], torch.empty_like(y)))
    steps_ = [TrainStep(model, opt, xb, sb, lens, yb, reducer) for (xb, sb, yb) in bufs]

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        steps_[0].eager()
    barrier()
    if args.gemm_census:
        _capi.GEMM_LOG = []
        steps_[0].eager()
        torch.cuda.synchronize()
        import collections

        tms = collections.defaultdict(float)
        cnt = collections.Counter()
        for key, s_, e_ in _capi.GEMM_LOG:
            tms[key] += s_.elapsed_time(e_)
            cnt[key] += 1
        tot = sum(tms.values())
        print(f"gemm total {tot:.3f} ms over {sum(cnt.values())} calls", file=sys.stderr)
        for k, v in sorted(tms.items(), key=lambda kv: -kv[1]):
            M_, N_, K_, b1, b2 = k[:5]
            tf = 2.0 * M_ * N_ * K_ * b1 * b2 * cnt[k] / (v / 1e3) / 1e12 if v > 0 else 0
            print(f"gemm {v:8.3f} ms {cnt[k]:3d}x {tf:7.1f} TF/s {k}", file=sys.stderr)
        _capi.GEMM_LOG = None

    census_log = None
    if args.op_census:
        torch.cuda.synchronize()
        _capi.OP_LOG = []
        steps_[0].eager()
        torch.cuda.synchronize()
        census_log, _capi.OP_LOG = _capi.OP_LOG, None

    # The SWA kernels are timed with CUDA events recorded on their launching
    # stream; in graph mode the event records are nodes of the captured step,
    # so the durations come from the timed replays themselves.
    timed_ops = {"kl_swa_fwd": [], "kl_swa_bwd": []}
    n_step = _capi.launch_count()
    steps_[0].eager()
    launches_per_step = _capi.launch_count() - n_step
    use_graph = not args.eager
    if use_graph:
        try:
            _capi.TIMED, _capi.TIMED_EXTERNAL = timed_ops, True
            steps_[0].capture(warmup=0)
        finally:
            _capi.TIMED, _capi.TIMED_EXTERNAL = None, False
        for st in steps_[1:]:
            st.capture(warmup=0)
        for _ in range(args.warmup):
            steps_[0]()
        barrier()

    if census_log is not None:
        graph_census(census_log, steps_[0], use_graph)

    # ---- device-timed region: inputs resident in HBM ----------------------
    if not use_graph:
        _capi.TIMED = timed_ops
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for _ in range(args.steps):
        steps_[0]()
    host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
    e1.record()
    barrier()
    launches = launches_per_step * args.steps
    clk = clocks.stop()
    _capi.TIMED = None
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B / (ms / 1e3)

    # ---- roofline of the dominant kernel: SWA (fwd + bwd) ------------------
    nsw = sum(1 for l in range(cfg.L) if model.seq_live()[l] and not model.flags[l].skip_self_attention)
    swa_ms = [s.elapsed_time(e) for (s, e) in timed_ops["kl_swa_fwd"][-nsw:]] if nsw else []
    swab_ms = [s.elapsed_time(e) for (s, e) in timed_ops["kl_swa_bwd"][-nsw:]] if nsw else []

    flags, live = model.flags, model.seq_live()
    fps = metrics.train_flops_per_sample(cfg, flags, live)
    fps_ref = metrics.train_flops_per_sample(cfg, flags, [True] * cfg.L, "reference")
    macs = metrics.model_macs(cfg, flags, live)
    burst, sustained, hbm, peak_kind = peaks()

    # ---- e2e through the public API with host buffers ----------------------
    e2e = None
    if not args.no_e2e:
        Xh = torch.from_numpy(Xn).to(dtype).pin_memory()
        Sh = [torch.from_numpy(s).to(dtype).pin_memory() for s in Sn]
        yh = torch.from_numpy(yn).pin_memory()
        loss_h = torch.empty(args.steps, dtype=torch.float32).pin_memory()
        h2d = Xh.numel() * 2 + sum(s.numel() * 2 for s in Sh) + yh.numel() * 4
        copy = torch.cuda.Stream()
        ready = [torch.cuda.Event(), torch.cuda.Event()]
        done = [torch.cuda.Event(), torch.cuda.Event()]

        def fetch(i):
            st = steps_[i % 2]
            with torch.cuda.stream(copy):
                if i >= 2:
                    copy.wait_event(done[i % 2])  # step i-2 (same buffers) has finished reading them
                st.X.copy_(Xh, non_blocking=True)
                for a_, b_ in zip(st.S, Sh):
                    a_.copy_(b_, non_blocking=True)
                st.labels.copy_(yh, non_blocking=True)
                ready[i % 2].record(copy)

        barrier()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record()
        fetch(0)
        for i in range(args.steps):
            if i + 1 < args.steps:
                fetch(i + 1)  # prefetch overlaps step i
            torch.cuda.current_stream().wait_event(ready[i % 2])
            loss = steps_[i % 2]()
            done[i % 2].record()
            loss_h[i].copy_(loss.detach(), non_blocking=True)
        f1.record()
        barrier()
        ems = f0.elapsed_time(f1) / args.steps
        t = torch.tensor([ems], device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ems = float(t.item())
        e2e = {"value": world * B / (ems / 1e3), "unit": "samples/s", "h2d_bytes_per_step": int(h2d),
               "d2h_bytes_per_step": 4, "ms_per_step": ems,
               "note": "pinned host batch -> HBM on a copy stream (double-buffered prefetch) + loss read back"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        workers = max(1, min(host_cores(), args.cpu_workers))
        try:
            rates = cpu_reference(cfg, workers, 1, rounds=1)
            cpu = {"value": rates[0], "unit": "samples/s", "cores": workers, "kind": "port",
                   "sample": f"{workers} samples (1 per forked single-thread worker), oracle float64 fwd+bwd "
                             f"of the same config (oracle/model.py; dense masked T x T attention as the reference)"}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "samples/s", "cores": workers, "kind": "port", "sample": f"failed: {exc}"}

    if rank != 0:
        return
    swa_flops = 4.0 * sum(metrics._support(ev.T, ev.w, ev.causal) for ev in cfg.events) * cfg.d * B
    n_swa_layers = sum(1 for l in range(cfg.L) if live[l] and not flags[l].skip_self_attention)
    fwd_avg = (sum(swa_ms) / len(swa_ms)) if swa_ms else None
    bwd_avg = (sum(swab_ms) / len(swab_ms)) if swab_ms else None
    roof = None
    if fwd_avg:
        # The banded attention core reads Q, K, V (B*T*3*H*d_h bf16) and
        # writes O (bf16) + LSE (fp32) once: at d_h = 64 its floor is HBM
        # (bytes / 6.5 TB/s) above the tensor floor (executed flops / peak),
        # so the roofline is the HBM one; the tensor numbers ride along.
        H_ = cfg.heads
        swa_bytes = float(sum(B * ev.T * (3 * cfg.d * 2 + cfg.d * 2 + H_ * 4) for ev in cfg.events))
        ach_gbs = swa_bytes / (fwd_avg / 1e3) / 1e9
        ach_tf = swa_flops / (fwd_avg / 1e3) / 1e12
        traffic = None
        try:  # dram__bytes_read.sum + dram__bytes_write.sum of the same kernel/shape (ncu --set full)
            prof = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                               "r1_swa3_ncu.json")))
            k = prof["kernels"].get("swa_fwd_tc3_kernel")
            if k and args.config == "c2" and B == 128:
                traffic = k["dram_bytes_per_launch"]
        except (OSError, ValueError, KeyError):
            pass
        roof = {"bound": "hbm", "kernel": "kl_swa_fwd (banded flash attention core, swa_fwd_tc3_kernel)",
                "achieved": ach_gbs, "peak": hbm, "unit": "GB/s", "frac": ach_gbs / hbm, "traffic": traffic,
                "algorithmic_bytes_per_launch": swa_bytes, "avg_launch_ms": fwd_avg,
                "tensor": {"achieved_tflops": ach_tf, "peak": burst, "frac": ach_tf / burst,
                           "algorithmic_flops_per_launch": swa_flops,
                           "floor_ms": {"hbm": swa_bytes / hbm / 1e6, "tensor": swa_flops / burst / 1e9}},
                "bwd_avg_launch_ms": bwd_avg, "launches_per_step": n_swa_layers,
                "share_of_step": (fwd_avg + (bwd_avg or 0)) * n_swa_layers / ms}
    achieved_tf = fps * value / world / 1e12
    line = {
        "metric": "kunlun_fwd_bwd_samples_per_s", "value": value, "unit": "samples/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": workload(args, cfg, B, world),
        "mfu": {"value": achieved_tf / burst, "vs": f"{peak_kind} bf16 burst {burst} TFLOP/s",
                "vs_sustained": achieved_tf / sustained, "vs_datasheet_2250": achieved_tf / 2250.0,
                "achieved_tflops_per_gpu": achieved_tf, "train_flops_per_sample": fps,
                "ledger": "executed matmul MACs x2 x3 (metrics.py), liveness-pruned, reassociated forms",
                "reference_formulation_flops_per_sample": fps_ref, "fwd_macs_by_part": macs},
        "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk, "host_issue_ms_per_step": host_ms, "cuda_graph": use_graph,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
