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

import os

# The CPU reference legs fork single-thread numpy workers: OpenBLAS must be
# single-threaded before numpy (imported by torch / the package) first loads
# it, or every forked worker spins a full-width BLAS pool (oversubscription).
for _v in ("OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

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

    try:  # in case BLAS was initialised multi-threaded before the env was set
        from threadpoolctl import threadpool_limits

        threadpool_limits(1)
    except Exception:
        pass
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


def oracle_spec(cfg, L=None):
    from oracle import model as OM

    return OM.ModelSpec(L=L or cfg.L, d=cfg.d, heads=cfg.heads, n_ctx=cfg.n_ctx, n_sum=cfg.n_sum, n_kv=cfg.n_kv,
                        experts=cfg.experts, compskip=cfg.compskip, gdpa_acts=tuple(cfg.gdpa_acts),
                        expert_hidden=cfg.expert_hidden, head_hidden=cfg.head_hidden,
                        events=[OM.EventSpec(T=e.T, w=e.w, budget=e.budget, n_seeds=e.n_seeds, rank=e.rank,
                                             causal=e.causal) for e in cfg.events])


def reference_layers(cfg):
    """Layers the CPU reference runs per sample: the whole model when that is
    cheap, else a layer sample (1 layer, or one even + one odd layer under
    CompSkip, whose layers alternate) scaled to cfg.L ("time
    per-layer on >= P samples and state the L-scaling explicitly")."""
    work = cfg.L * sum(e.T for e in cfg.events) * cfg.d * cfg.d
    if work <= 4 * 1024 * 256 * 256:  # c1, c2: the full model
        return cfg.L
    return min(cfg.L, 2 if cfg.compskip else 1)


def cpu_reference(cfg, workers: int, samples_per_worker: int = 1, rounds: int = 1, warm: int = 0):
    """Times the float64 oracle fwd+bwd (the reference algorithm restated,
    oracle/model.py) with ``workers`` forked single-thread processes, each on
    ``samples_per_worker`` samples per round.  Returns (per-round samples/s
    of the FULL model, layers run per sample); with a layer sample the rate is
    scaled by layers_run / cfg.L."""
    import multiprocessing as mp

    from oracle import model as OM

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    Lr = reference_layers(cfg)
    spec = oracle_spec(cfg, Lr)
    _CPU_STATE["spec"] = (spec, OM.init_params(spec, seed=0))
    ctx = mp.get_context("fork")
    rates = []
    with ctx.Pool(workers) as pool:
        for r in range(warm + rounds):
            t0 = time.perf_counter()
            done = sum(pool.map(_cpu_worker, [("spec", samples_per_worker, 1000 * r + i) for i in range(workers)]))
            dt = time.perf_counter() - t0
            if r >= warm:
                rates.append(done / dt * Lr / cfg.L)
    return rates, Lr


def cpu_model_name():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
    rates, Lr = cpu_reference(cfg, workers, 1, rounds=args.steps, warm=args.warmup)
    v = statistics.median(rates)
    sample = (f"{workers} samples/step (1 per forked single-thread worker), oracle float64 fwd+bwd of "
              + ("the full model" if Lr == cfg.L else f"{Lr} of {cfg.L} layers, rate scaled by {Lr}/{cfg.L}")
              + f"; host CPU {cpu_model_name()}")
    line = {
        "impl": "reference", "metric": "kunlun_fwd_bwd_samples_per_s", "value": v, "unit": "samples/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000.0 * workers / v,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": workload(args, cfg, B, world),
        "cpu_baseline": {"value": v, "unit": "samples/s", "cores": workers, "kind": "port", "sample": sample},
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


NCU_KERNELS = {  # roofline family -> kernel-name substrings (CUPTI / ncu names)
    "gemm": ("gemm_tc_kernel", "gemm_simt_kernel", "splitk_reduce"),
    "swa_fwd": ("swa_fwd_tc", "swa_fwd_kernel"), "swa_bwd": ("swa_bwd_", "swa_rowdot"),
    "gdpa_fwd": ("gdpa_fwd",), "gdpa_bwd": ("gdpa_bwd",), "hsp_fwd": ("hsp_fwd",),
    "hsp_bwd": ("hsp_bwd",), "colsoftmax_fwd": ("colsoftmax_fwd_kernel",),
    "colsoftmax_bwd": ("colsoftmax_bwd_kernel",), "adam": ("adam_kernel",),
}


def family_of(kernel_name):
    for f, subs in NCU_KERNELS.items():
        if any(x in kernel_name for x in subs):
            return f
    return None


def kernel_records(step):
    """[(kernel name, device us)] of one replay of ``step`` (CUPTI)."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        step()
        torch.cuda.synchronize()
    return [(e.name, e.time_range.end - e.time_range.start) for e in prof.events()
            if e.device_type.name == "CUDA"]


def _ncu_traffic(config, B):
    """{family: {"dram_bytes_per_launch", "tensor_pipe_pct", ...}} from the
    committed ncu --set full summary of this config (profiles/ncu_<config>_B<B>.json,
    written by profiles/summarize_ncu.py), or {}."""
    try:
        with open(os.path.join(ROOT, "profiles", f"ncu_{config}_B{B}.json")) as f:
            return json.load(f).get("families", {})
    except (OSError, ValueError):
        return {}


def roofline_table(work, kernels, ms_step, burst, sustained, hbm, peak_kind, config, B):
    """Per kernel family of one step: launches and summed device time (CUPTI
    records of a replay of the captured step), the algorithmic flops / bytes
    the step's C-ABI calls declare (_capi._work_of), the bound (tensor when
    flops/bytes >= the ridge of the measured peaks), the achieved rate against
    the measured peak (sustained bf16: these kernels run inside a long step),
    and the ncu DRAM traffic where a capture exists.  ``share_of_step`` is the
    family's summed kernel time over the step time (branches overlap, so
    shares can sum past 1).  The headline ``roofline`` is the family with the
    most device time."""
    ridge = sustained * 1e12 / (hbm * 1e9)
    fam = {}
    for f, flops, nbytes, _, _ in work:
        d = fam.setdefault(f, {"launches": 0, "ms": 0.0, "flops": 0.0, "bytes": 0.0, "calls": 0, "tflops": 0.0})
        d["calls"] += 1
        d["flops"] += flops
        d["bytes"] += nbytes
        if flops >= ridge * nbytes:
            d["tflops"] += flops  # flops of calls that are tensor-bound on their own
    other = 0.0
    for name, us in kernels:
        f = family_of(name)
        if f is None or f not in fam:
            other += us / 1e3
            continue
        fam[f]["launches"] += 1
        fam[f]["ms"] += us / 1e3
    ncu = _ncu_traffic(config, B)
    table = {}
    for f, d in fam.items():
        if not d["launches"]:
            continue
        sec = d["ms"] / 1e3
        # a family is tensor-bound when most of its flops come from calls whose
        # own flops/bytes sit above the ridge (the GEMM family mixes K = d
        # projections with small per-sample products)
        tensor = d["flops"] > 0 and d["tflops"] >= 0.5 * d["flops"]
        gbs, tfs = d["bytes"] / sec / 1e9, d["flops"] / sec / 1e12
        ach, peak, unit = (tfs, sustained, "TFLOP/s") if tensor else (gbs, hbm, "GB/s")
        n = d["launches"]
        table[f] = {"bound": "tensor" if tensor else "hbm", "achieved": ach, "peak": peak, "unit": unit,
                    "frac": ach / peak, "launches": n, "calls": d["calls"], "avg_launch_ms": d["ms"] / n,
                    "ms_per_step": d["ms"], "share_of_step": d["ms"] / ms_step,
                    "algorithmic_flops_per_launch": d["flops"] / n, "algorithmic_bytes_per_launch": d["bytes"] / n,
                    "achieved_gbs": gbs, "achieved_tflops": tfs, "tensor_bound_flop_share": d["tflops"] / max(d["flops"], 1.0),
                    "traffic": None}
        nc = ncu.get(f)
        if nc:
            table[f]["traffic"] = nc.get("dram_bytes_per_launch")
            table[f]["ncu"] = nc
    if not table:
        return table, None
    table["_other_kernels"] = {"ms_per_step": other, "share_of_step": other / ms_step}
    top = max((k for k in table if not k.startswith("_")), key=lambda k: table[k]["ms_per_step"])
    t = table[top]
    roof = {"bound": t["bound"], "kernel": top, "achieved": t["achieved"], "peak": t["peak"], "unit": t["unit"],
            "frac": t["frac"], "traffic": t["traffic"],
            "peak_kind": f"{peak_kind} " + ("bf16 sustained" if t["bound"] == "tensor" else "HBM copy"),
            "algorithmic_per_launch": t["algorithmic_flops_per_launch" if t["bound"] == "tensor"
                                        else "algorithmic_bytes_per_launch"],
            "avg_launch_ms": t["avg_launch_ms"], "launches_per_step": t["launches"],
            "share_of_step": t["share_of_step"]}
    return table, roof


def workload(args, cfg, B, world):
    ev = cfg.events[0]
    abl = f"_ablation_{args.ablation.replace(',', '+')}" if args.ablation else ""
    return {"workload": f"kunlun_{args.config}{abl}_train_step", "model": "kunlun", "layers": cfg.L, "d": cfg.d,
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
    ap.add_argument("--config", default="c4", help="BASELINE.json configs: c4 (the 1/2/4/8-GPU DP config, default), "
                    "c1, c2, c3")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--ablation", default="", help="PAPER.md Table 2 switch: pffn (pffn_original instead of GDPA), "
                    "pma (PMA summaries instead of HSP), full (full attention instead of SWA); comma-separated")
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

    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # --gpus N without a launcher: one process per GPU via torchrun (NCCL)
        import random

        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={random.randint(20000, 40000)}",
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))

    world = int(os.environ.get("WORLD_SIZE", "1"))
    if args.gpus > 1 and world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    from paper_2602_10016_b200.configs import CONFIGS

    cfg, B = CONFIGS[args.config]()
    if args.batch:
        B = args.batch
    for a in filter(None, args.ablation.split(",")):
        if a not in ("pffn", "pma", "full"):
            raise SystemExit(f"unknown ablation {a!r}")
        setattr(cfg, {"pffn": "pffn", "pma": "summarizer", "full": "attention"}[a],
                {"pffn": "original", "pma": "pma", "full": "full"}[a])

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
    if model.groups is not None:  # grouped event types: the sequences as adjacent slices of one batch
        from paper_2602_10016_b200.grouped import stage

        S, lens = stage(S), stage(lens)

    from paper_2602_10016_b200.optim import TrainStep

    bufs = [(X, S, y)]
    if not args.no_e2e:  # a second static input set: the e2e loop double-buffers host->device copies
        bufs.append((torch.empty_like(X), list(torch.empty((len(S),) + tuple(S[0].shape), device=dev, dtype=dtype)
                                               .unbind(0)) if model.groups is not None
                     else [torch.empty_like(s) for s in S], torch.empty_like(y)))
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
    # Per-launch work accounting (roofline table): every accounted launch of
    # one step is bracketed by external CUDA events recorded on its launching
    # stream; in graph mode they are nodes of the captured step, so the
    # durations come from the timed replays themselves.
    n_step = _capi.launch_count()
    work = []  # (family, algorithmic flops, bytes) of every accounted launch of one step
    _capi.WORK, _capi.WORK_EVENTS = work, False
    try:
        steps_[0].eager()
    finally:
        _capi.WORK, _capi.WORK_EVENTS = None, True
    launches_per_step = _capi.launch_count() - n_step
    use_graph = not args.eager
    if use_graph:
        steps_[0].capture(warmup=0)
        for st in steps_[1:]:
            st.capture(warmup=0)
        for _ in range(args.warmup):
            steps_[0]()
        barrier()

    if census_log is not None:
        graph_census(census_log, steps_[0], use_graph)

    # ---- device-timed region: inputs resident in HBM ----------------------
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    h0 = time.perf_counter()
    for i in range(args.steps):
        steps_[0]()
    host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
    e1.record()
    barrier()
    launches = launches_per_step * args.steps
    clk = clocks.stop()
    steps_[0].check_numerics()  # NumericsError if any timed step produced a NaN / Inf logit or loss
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    value = world * B / (ms / 1e3)

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
            rates, Lr = cpu_reference(cfg, workers, 1, rounds=1)
            cpu = {"value": rates[0], "unit": "samples/s", "cores": workers, "kind": "port",
                   "sample": f"{workers} samples (1 per forked single-thread worker), oracle float64 fwd+bwd "
                             f"of the same config (oracle/model.py: the reference's masked attention, block-banded "
                             f"above T=1024)" + ("" if Lr == cfg.L else f", {Lr} of {cfg.L} layers, rate scaled by "
                                                                      f"{Lr}/{cfg.L}")
                             + f"; host CPU {cpu_model_name()}"}
        except Exception as exc:  # pragma: no cover
            cpu = {"value": None, "unit": "samples/s", "cores": workers, "kind": "port", "sample": f"failed: {exc}"}

    if rank != 0:
        return
    # ---- per-kernel-family roofline table (after, and outside, the timed
    # regions): CUPTI kernel records of one more replay of the same captured
    # step (torch.profiler), grouped by kernel family, against the
    # algorithmic work the C-ABI calls of one step declare.
    table, roof = None, None
    if rank == 0:
        table, roof = roofline_table(work, kernel_records(steps_[0]), ms, burst, sustained, hbm, peak_kind,
                                     args.config, B)
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
        "roofline": roof, "roofline_table": table, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches),
        "clocks": clk, "host_issue_ms_per_step": host_ms, "cuda_graph": use_graph,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
