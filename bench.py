"""Benchmark: one learned-optimizer step over ViT-B/16-shaped parameters.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A "step" is LearnedOptimizer.step() over all 152 ViT-B/16 tensors (86,567,656
f32 parameters) with synthetic gradients already resident in HBM: factor pass,
feature-statistics pass, apply pass (state advance, features, MLP, update,
decoupled decay).  Metric: parameters stepped per second (Gparams/s,
higher is better), whole job.  Under torchrun (N > 1) the step is sharded by
element ranges across ranks (paper_2506_10315_b200.dist); the time is the max
over ranks.

Also reported on the same line:
  e2e          the same step through the public API with HOST buffers: each
               step copies the gradients from pinned host memory and reads the
               updated parameters back, both inside the timed region;
  roofline     the dominant kernel (apply pass) against measured HBM bandwidth,
               44 algorithmic bytes per parameter;
  cpu_baseline the CPU oracle (oracle/, a bitwise restatement of the
               reference) on a bounded sample, all host cores;
  velo         the same measurement for the VeLO-MLP feature set;
  clocks       nvidia-smi SM clocks and throttle reasons sampled during timing.

`--impl reference` times the reference algorithm on the host cores instead
(the oracle port, OpenMP over tensors) on a bounded sample of the same
workload, with the same metric/unit.
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

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

ALGO_BYTES_PER_PARAM = 44          # read theta,g,M1..3,V; write theta,M1..3,V
HBM_PEAK_FALLBACK = 6650.0         # GB/s, B200_PROFILING.md fallback


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": HBM_PEAK_FALLBACK}, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._thr = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.samples.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:  # noqa: BLE001
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._thr.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for s in self.samples for k in range(4)
                          if len(s) > 3 + k and s[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


def dist_setup(args):
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist

        # LOPT_DIST_BACKEND=gloo with LOPT_SHARE_GPU=1 runs all ranks on cuda:0
        # (a functional check of the multi-rank path on a one-GPU box)
        backend = os.environ.get("LOPT_DIST_BACKEND", "nccl")
        dev = 0 if os.environ.get("LOPT_SHARE_GPU") else local
        torch.cuda.set_device(dev)
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
        else:
            dist.init_process_group(backend)
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def make_model(workload, device, seed=0):
    import torch

    from paper_2506_10315_b200.workloads import WORKLOADS

    g = torch.Generator(device="cpu").manual_seed(seed)
    params, grads = [], []
    for _, shape in WORKLOADS[workload]():
        p = torch.empty(shape, dtype=torch.float32)
        fan_in = int(np.prod(shape[1:])) if len(shape) > 1 else 1
        p.normal_(0.0, 1.0 / max(1.0, fan_in) ** 0.5, generator=g)
        params.append(torch.nn.Parameter(p.to(device)))
        gr = torch.empty(shape, dtype=torch.float32)
        gr.normal_(0.0, 1e-3, generator=g)
        grads.append(gr.to(device))
    return params, grads


def workload_hparams(workload):
    """BASELINE.json config 5: GPT-2 medium runs with a cosine LR schedule and
    weight decay 0.01; the others at constant lr 1, no decay.
    (Same kernels either way: decay is one multiply, the schedule a host scalar.)"""
    if workload == "gpt2_medium":
        from paper_2506_10315_b200 import ScheduleConfig

        return {"weight_decay": 0.01,
                "schedule": ScheduleConfig(kind="cosine", max_lr=1.0, min_lr=0.1,
                                           warmup_steps=2, total_steps=10_000)}
    return {}


def build_optimizer(params, feature_set, mode, world, strategy="range", hp=None):
    """feature_set "velo" is the full VeLO optimizer (VELO_MLP features + the
    per-tensor LSTM hypernetwork mixing a bank of MLPs); "small_fc_lopt" and
    "velo_mlp" are the single-MLP learned optimizers."""
    hp = hp or {}
    # N > 1: the parameter exchange is fused into the apply kernel (stores to
    # the peers' IPC-mapped arenas over NVLink) unless LOPT_GATHER=nccl
    gather = os.environ.get("LOPT_GATHER", "p2p" if mode == "fast" else "nccl")
    if feature_set == "velo":
        if world > 1:
            from paper_2506_10315_b200.dist import ShardedVeLO

            try:
                return ShardedVeLO(params, mode=mode, check_errors=False, gather=gather,
                                   strategy=strategy, **hp)
            except Exception as e:  # noqa: BLE001
                if "LOPT_GATHER" in os.environ:
                    raise   # an explicitly requested exchange is not substituted
                print(f"bench: p2p gather unavailable ({e}); NCCL all-gather", file=sys.stderr)
                opt = ShardedVeLO(params, mode=mode, check_errors=False, strategy=strategy, **hp)
                opt.gather_fallback = f"p2p unavailable: {e}"[:200]
                return opt
        from paper_2506_10315_b200.velo import VeLO_CUDA

        return VeLO_CUDA(params, mode=mode, check_errors=False, **hp)
    if world > 1:
        from paper_2506_10315_b200.dist import ShardedLearnedOptimizer

        try:
            return ShardedLearnedOptimizer(params, feature_set=feature_set, mode=mode,
                                           check_errors=False, gather=gather, strategy=strategy,
                                           **hp)
        except Exception as e:  # noqa: BLE001
            if "LOPT_GATHER" in os.environ:
                raise   # an explicitly requested exchange is not substituted
            print(f"bench: p2p gather unavailable ({e}); NCCL all-gather", file=sys.stderr)
            opt = ShardedLearnedOptimizer(params, feature_set=feature_set, mode=mode,
                                          check_errors=False, strategy=strategy, **hp)
            opt.gather_fallback = f"p2p unavailable: {e}"[:200]
            return opt
    from paper_2506_10315_b200 import LearnedOptimizer

    return LearnedOptimizer(params, feature_set=feature_set, mode=mode, check_errors=False, **hp)


def step_kwargs(opt):
    """VeLO's step takes the training loss; a fixed synthetic one."""
    return {"loss": 2.3} if hasattr(opt, "hypernet") else {}


def time_device(opt, params, grads, steps, warmup, world):
    """Device-resident inputs; CUDA events on the current stream.  The timed
    steps are plain optimizer.step() calls (one graph launch each on one
    device).  On one device they also record their own phase events (event
    nodes inside the captured graph); a sharded step (Python between its
    phases and collectives) records phases in a second pass instead, so the
    headline loop carries no per-phase host work."""
    import torch

    for p, g in zip(params, grads):
        p.grad = g
    kw = step_kwargs(opt)
    # the timed steps record their own phase events (inside the captured graph
    # on one device), so the phase times -- the roofline's apply duration --
    # come from the measured steps themselves; warm-up captures that graph
    inline_phases = world == 1
    opt.phase_events = [] if inline_phases else None
    for _ in range(warmup):
        opt.step(**kw)
    torch.cuda.synchronize()
    barrier(world)
    torch.cuda.synchronize()
    opt.phase_events = [] if inline_phases else None
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    start.record()
    marks[0].record()
    for k in range(steps):
        opt.step(**kw)
        marks[k + 1].record()
    end.record()
    torch.cuda.synchronize()
    barrier(world)
    ms = start.elapsed_time(end)
    if not inline_phases:
        opt.phase_events = []
        for _ in range(steps):
            opt.step(**kw)
        torch.cuda.synchronize()
    phases = {}
    for name, a, b in opt.phase_events:
        phases.setdefault(name, []).append(a.elapsed_time(b))
    opt.phase_events = None
    # host enqueue cost per step (no sync inside), plain steps
    for _ in range(2):
        opt.step(**kw)
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    for _ in range(steps):
        opt.step(**kw)
    host_ms = (time.perf_counter() - h0) * 1e3 / steps
    torch.cuda.synchronize()
    barrier(world)
    per_step = sorted(marks[k].elapsed_time(marks[k + 1]) for k in range(steps))
    if world > 1 and hasattr(opt, "set_exchange"):
        # the same step without the parameter exchange
        opt.set_exchange(False)
        for _ in range(2):
            opt.step(**kw)
        torch.cuda.synchronize()
        barrier(world)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record()
        for _ in range(steps):
            opt.step(**kw)
        s1.record()
        torch.cuda.synchronize()
        barrier(world)
        opt.set_exchange(True)
        phases["_no_exchange_ms"] = max_over_ranks(s0.elapsed_time(s1), world) / steps
    q = lambda f: per_step[min(len(per_step) - 1, int(f * (len(per_step) - 1) + 0.5))]  # noqa: E731
    phases["_step_quantiles"] = [q(0.1), q(0.5), q(0.9)]
    phases["_host_ms"] = host_ms
    launches = sum(pl.launches_last_step() for pl in opt.plans())
    return max_over_ranks(ms, world), phases, launches


# tensor groups of the host-buffer step: finer groups shorten the pipeline's
# fill (first upload) and drain (last download); with double-buffered gradient
# arenas 8 and 16 measure alike (8.0 ms), 32 is host-launch bound (9.8 ms)
E2E_CHUNKS = int(os.environ.get("LOPT_E2E_CHUNKS", "8"))


def time_e2e(opt, params, grads, steps, warmup, world):
    """Public-API step with host buffers: the gradients come from pinned host
    memory and the updated parameters go back to pinned host memory, both
    inside the timed region, every step.  Single GPU: LearnedOptimizer.step_host
    (chunked, H2D / step / D2H overlapped on separate streams); sharded: the
    plain copies around step()."""
    import torch

    # host buffers as one pinned block each, tensors as consecutive views (how
    # a host-resident caller that owns its arrays would lay them out); the
    # step then moves every tensor group as one PCIe copy
    sizes = [g.numel() for g in grads]
    offs = np.cumsum([0] + sizes)
    g_block = torch.empty(int(offs[-1]), dtype=torch.float32).pin_memory()
    p_block = torch.empty(int(offs[-1]), dtype=torch.float32).pin_memory()
    host_g, host_p = [], []
    for k, (g, p) in enumerate(zip(grads, params)):
        g_block[offs[k]:offs[k + 1]].copy_(g.reshape(-1))
        host_g.append(g_block[offs[k]:offs[k + 1]].view(g.shape))
        host_p.append(p_block[offs[k]:offs[k + 1]].view(p.shape))
    dev_g = [torch.empty_like(g) for g in grads]
    for p, g in zip(params, dev_g):
        p.grad = g
    piped = world == 1 and hasattr(opt, "step_host")
    # sharded (element ranges, one bucket): each rank's process uploads the
    # gradient of its own slice and downloads its own slice of the result --
    # one copy each way, the slices of all ranks together cover the model
    sliced = (world > 1 and getattr(opt, "slice_len", None) is not None
              and getattr(opt, "strategy", "range") == "range")
    h2d = sum(g.numel() * 4 for g in grads)
    d2h = sum(p.numel() * 4 for p in params)
    if sliced:
        import torch.distributed as dist

        fg = opt.flat_grads()
        S, rank = opt.slice_len, dist.get_rank()
        lo, hi = min(rank * S, int(offs[-1])), min((rank + 1) * S, int(offs[-1]))

    chunks = E2E_CHUNKS

    def one():
        if piped:
            opt.step_host(host_g, host_p, chunks=chunks)
            return
        if sliced:
            fg[lo:hi].copy_(g_block[lo:hi], non_blocking=True)
            opt.step()
            p_block[lo:hi].copy_(opt.flat[lo:hi], non_blocking=True)
            return
        for d, h in zip(dev_g, host_g):
            d.copy_(h, non_blocking=True)
        opt.step()
        for h, p in zip(host_p, params):
            h.copy_(p.detach(), non_blocking=True)

    for _ in range(warmup):
        one()
    torch.cuda.synchronize()
    barrier(world)
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    start.record()
    for _ in range(steps):
        one()
    end.record()
    torch.cuda.synchronize()
    barrier(world)
    return max_over_ranks(start.elapsed_time(end), world), h2d, d2h


_INPUTS = {}


def run_cpu_oracle(workload, feature_set, budget_params, steps, warmup, threads=0):
    """The oracle port on a bounded prefix of the workload (census order),
    with the GPU arm's synthetic inputs (_ref_inputs)."""
    from oracle import oracle as O

    kind = O.KIND_BY_NAME[feature_set]
    if workload not in _INPUTS:
        _INPUTS[workload] = _ref_inputs(workload)
    P0, G0 = _INPUTS[workload]
    idx, total = [], 0
    for j, p in enumerate(P0):   # keep the workload's mix: walk in order, skip what overflows
        if total + p.size <= budget_params:
            idx.append(j)
            total += p.size
    params = [P0[j].copy() for j in idx]
    grads = [G0[j] for j in idx]
    states = [O.OState.zeros(*p.shape) for p in params]
    w = O.random_weights(39 if kind == O.SMALL_FC_LOPT else 29, seed=0)
    for _ in range(warmup):
        O.opt_step(params, states, grads, w, kind, 1.0, threads=threads)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.opt_step(params, states, grads, w, kind, 1.0, threads=threads)
        times.append(time.perf_counter() - t0)
    cores = threads if threads > 0 else len(os.sched_getaffinity(0))
    return {"params": total, "tensors": len(idx), "step_s": statistics.median(times),
            "cores": cores, "steps": steps}


REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def shipped_reference_available():
    """The unmodified reference package installed into baseline/_ref (pip
    --target)."""
    return os.path.isdir(os.path.join(REF_DIR, "lopt"))


def _ref_inputs(workload, seed=0):
    """The GPU arm's synthetic inputs (make_model, same generator and seed) as
    2-D NumPy arrays -- identical bytes on both arms."""
    from paper_2506_10315_b200 import view_2d

    params, grads = make_model(workload, "cpu", seed=seed)
    P = [p.detach().numpy().reshape(view_2d(p.shape)) for p in params]
    G = [g.numpy().reshape(view_2d(g.shape)) for g in grads]
    return P, G


def _ref_handle(lo, P, idx, feature_set):
    w = lo.engine.random_weights(39 if feature_set == "small_fc_lopt" else 29, seed=0)
    spec = (lo.features.small_fc_lopt_spec() if feature_set == "small_fc_lopt"
            else lo.features.velo_mlp_spec())
    return lo.optim.OptimizerHandle.fresh([(f"t{j}", P[j].copy()) for j in idx], w, spec)


def _ref_proc(conn, idx, feature_set):
    """Pool worker: the unmodified reference opt_step on its whole tensors."""
    import lopt as lo
    import lopt.engine  # noqa: F401
    import lopt.features  # noqa: F401
    import lopt.optim  # noqa: F401

    h = _ref_handle(lo, _REF_P, idx, feature_set)
    g = [_REF_G[j] for j in idx]
    while conn.recv():
        t0 = time.perf_counter()
        lo.optim.opt_step(h, g)
        conn.send(time.perf_counter() - t0)


_REF_P = _REF_G = None


def run_shipped_reference(workload, feature_set, steps, warmup, time_budget_s=120.0):
    """the shipped reference's opt_step (numba, fused
    path, lr 1) on the GPU arm's inputs -- (ii) all host cores: P forked
    processes each stepping a disjoint whole-tensor subset (greedy largest
    first, distsim.py:109-118); tensors are independent, so the results are
    those of one opt_step -- and (i) one process on one core.  The per-step
    sample is the largest-first prefix of the census that keeps the whole
    --steps/--warmup run inside `time_budget_s`."""
    import multiprocessing as mp

    global _REF_P, _REF_G
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    import lopt as lo
    import lopt.engine  # noqa: F401
    import lopt.features  # noqa: F401
    import lopt.optim  # noqa: F401

    if workload not in _INPUTS:
        _INPUTS[workload] = _ref_inputs(workload)
    P, G = _INPUTS[workload]
    # JIT-compile in the parent so the forked workers inherit the machine code
    hw = _ref_handle(lo, [P[0][:2, :16].copy(), P[1][:8].copy()], [0, 1], feature_set)
    lo.optim.opt_step(hw, [G[0][:2, :16].copy(), G[1][:8].copy()])
    # (i) one process: the largest-first prefix up to ~3 M params, one step
    sizes = [p.size for p in P]
    one, tot = [], 0
    for j in sorted(range(len(P)), key=lambda j: -sizes[j]):
        if tot + sizes[j] <= 3_000_000:
            one.append(j)
            tot += sizes[j]
    h1 = _ref_handle(lo, P, one, feature_set)
    t0 = time.perf_counter()
    lo.optim.opt_step(h1, [G[j] for j in one])
    t_one = time.perf_counter() - t0
    rate1 = tot / t_one
    del h1
    # (ii) all cores
    cores = len(os.sched_getaffinity(0))
    est_rate = rate1 * cores * 0.8
    budget = time_budget_s / (steps + warmup) * est_rate
    chosen, total = [], 0
    for j in sorted(range(len(P)), key=lambda j: -sizes[j]):
        if total + sizes[j] <= max(budget, sizes[j] if not chosen else 0):
            chosen.append(j)
            total += sizes[j]
    loads = [[0, []] for _ in range(cores)]
    for j in chosen:                       # greedy largest-first (distsim.make_plan)
        b = min(loads, key=lambda x: x[0])
        b[0] += sizes[j]
        b[1].append(j)
    _REF_P, _REF_G = P, G
    ctx = mp.get_context("fork")
    pipes, procs = [], []
    for _, idx in loads:
        if not idx:
            continue
        a, b = ctx.Pipe()
        pr = ctx.Process(target=_ref_proc, args=(b, idx, feature_set), daemon=True)
        pr.start()
        pipes.append(a)
        procs.append(pr)
    times = []
    try:
        for k in range(warmup + steps):
            t0 = time.perf_counter()
            for a in pipes:
                a.send(True)
            for a in pipes:
                a.recv()
            if k >= warmup:
                times.append(time.perf_counter() - t0)
    finally:
        for a in pipes:
            a.send(False)
        for pr in procs:
            pr.join(timeout=10)
    return {"params": total, "tensors": len(chosen), "step_s": statistics.median(times),
            "cores": len(procs), "single": {"params": tot, "tensors": len(one), "step_s": t_one}}


def cpu_reference(args, n_params, steps, warmup, time_budget_s=120.0):
    """The CPU baseline of both arms: the shipped reference (baseline/_ref,
    numba opt_step, all host cores as a process pool) when installed, with the
    oracle port (oracle/, OpenMP over tensors) timed beside it; else the port
    alone.  Returns (value Gparams/s, ms per step, cpu_baseline dict)."""
    if shipped_reference_available() and not os.environ.get("LOPT_REF_PORT"):
        r = run_shipped_reference(args.workload, args.feature_set, steps, warmup, time_budget_s)
        value = r["params"] / r["step_s"] / 1e9
        s1 = r["single"]
        rp = run_cpu_oracle(args.workload, args.feature_set, n_params, 1, 1)
        base = {"value": value, "unit": "Gparams/s", "cores": r["cores"], "kind": "reference",
                "sample": (f"{r['tensors']} of the {args.workload} tensors / {r['params']} params "
                           f"(largest-first prefix within the time budget), the shipped "
                           f"reference (baseline/_ref lopt.optim.opt_step, path='fused', numba) "
                           f"in {r['cores']} forked processes over disjoint whole-tensor "
                           f"subsets (greedy largest-first), median of {steps} steps"),
                "single_process": {"value": s1["params"] / s1["step_s"] / 1e9,
                                   "unit": "Gparams/s", "cores": 1,
                                   "sample": f"{s1['tensors']} largest tensors / {s1['params']} "
                                             f"params, one opt_step"},
                "port": {"value": rp["params"] / rp["step_s"] / 1e9, "unit": "Gparams/s",
                         "cores": rp["cores"], "kind": "port",
                         "sample": "the whole workload, oracle/ (bitwise restatement, 64-lane "
                                   "blocked MLP like engine.py:441-480, OpenMP over tensors), "
                                   "one step"}}
        return value, r["step_s"] * 1e3, base
    budget = int(max(1_000_000, min(args.cpu_budget or n_params, n_params * 40 // (steps + 1))))
    r = run_cpu_oracle(args.workload, args.feature_set, budget, steps, warmup)
    value = r["params"] / r["step_s"] / 1e9
    base = {"value": value, "unit": "Gparams/s", "cores": r["cores"], "kind": "port",
            "sample": (f"{r['tensors']} of the {args.workload} tensors, {r['params']} params "
                       f"(largest-first prefix of the census), oracle/ (bitwise restatement of "
                       f"the reference, OpenMP over tensors), median of {r['steps']} steps")}
    r1 = run_cpu_oracle(args.workload, args.feature_set, 3_000_000, 1, 0, threads=1)
    base["single_process"] = {"value": r1["params"] / r1["step_s"] / 1e9, "unit": "Gparams/s",
                              "cores": 1, "sample": f"{r1['tensors']} tensors / {r1['params']} "
                                                    f"params, one step"}
    return value, r["step_s"] * 1e3, base


def reference_arm(args, world, rank):
    """--impl reference: the reference on the host cores (cpu_reference), same
    metric, config and synthetic inputs as the GPU arm; rank 0 only."""
    if rank != 0:
        return
    from paper_2506_10315_b200.workloads import census

    n_tensors, n_params = census(args.workload)
    hp = workload_hparams(args.workload)
    value, ms, base = cpu_reference(args, n_params, args.steps, args.warmup)
    line = {
        "impl": "reference", "metric": metric_name(args), "value": value, "unit": "Gparams/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 else "none",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(args, hp, n_tensors, n_params, world),
        "cpu_baseline": base,
        "e2e": {"value": value, "unit": "Gparams/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def bench_config(args, hp, n_tensors, n_params, world):
    """The workload description shared by both arms (same keys and values)."""
    return {"workload": args.workload, "feature_set": args.feature_set,
            "hparams": ({k: (repr(v) if k == "schedule" else v) for k, v in hp.items()}
                        or {"lr": 1.0, "weight_decay": 0.0}),
            "tensors": n_tensors, "params": n_params,
            "parallelism": (("element-sharded" if args.strategy == "range" else
                             "tensor-owner-sharded") + f" x{world}") if world > 1 else "single",
            "l2": f"inputs larger than L2 (each f32 array {n_params * 4 / 1e6:.0f} MB > 126 MB)"}


METRIC = "optimizer step ms + Gparams/s at ViT-B/16 (small_fc_lopt, VeLO) vs roofline"


def metric_name(args):
    return METRIC


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="vit_b16")
    ap.add_argument("--feature-set", default="small_fc_lopt")
    ap.add_argument("--mode", default=os.environ.get("LOPT_BENCH_MODE", "fast"),
                    help="fast (tensor-core product path, fp32 tolerance) or strict (bitwise)")
    ap.add_argument("--cpu-budget", type=int, default=0,
                    help="params in the bounded CPU sample (0: the whole workload)")
    ap.add_argument("--strategy", default=os.environ.get("LOPT_SHARD_STRATEGY", "range"),
                    choices=["range", "owner"],
                    help="N>1: element ranges (REDUCE_SCATTER) or whole tensors per owner (FSDP_A2A)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-velo", action="store_true")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)

    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        reference_arm(args, world, rank)
        return
    import torch

    from paper_2506_10315_b200.workloads import census

    n_tensors, n_params = census(args.workload)
    peaks, peak_kind = measured_peaks()
    hbm_peak = float(peaks.get("hbm_gbs", HBM_PEAK_FALLBACK))
    dev = torch.device("cuda", torch.cuda.current_device())
    params, grads = make_model(args.workload, dev, seed=0)

    hp = workload_hparams(args.workload)
    opt = build_optimizer(params, args.feature_set, args.mode, world, args.strategy, hp)
    gather_used = getattr(opt, "gather", "nccl")
    gather_fallback = getattr(opt, "gather_fallback", None)
    clk = ClockSampler(torch.cuda.current_device())
    clk.__enter__()   # sampled through the timed steps, the phase pass and the e2e run
    ms, phases, launches = time_device(opt, params, grads, args.steps, args.warmup, world)
    value = n_params * args.steps / (ms / 1e3) / 1e9
    apply_ms = statistics.mean(phases.get("apply", [float("nan")]))
    local_params = sum(pl.local_elements() for pl in opt.plans())
    achieved = ALGO_BYTES_PER_PARAM * local_params / (apply_ms / 1e3) / 1e9
    quant = phases.pop("_step_quantiles", None)
    no_exchange_ms = phases.pop("_no_exchange_ms", None)
    host_ms = phases.pop("_host_ms", None)
    roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": None, "kernel": "apply (phase 2)",
                "peak_source": peak_kind, "frac_vs_8tbs_spec": achieved / 8000.0,
                "phase_ms": {k: statistics.mean(v) for k, v in phases.items()},
                "step_frac_of_roofline": (ALGO_BYTES_PER_PARAM * n_params / (ms / args.steps / 1e3)
                                          / 1e9) / hbm_peak}
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                t = json.load(f)
            key = f"{args.workload}/{args.feature_set}/{args.mode}"
            if key in t:
                # DRAM bytes (read + write) of one apply launch from the committed
                # ncu capture, against ALGO_BYTES_PER_PARAM * params algorithmic
                roofline["traffic"] = t[key]["bytes"]
                roofline["traffic_unit"] = "GB per launch (ncu dram__bytes_read+write)"
                if "step_bytes" in t[key]:
                    # every kernel of the step (factor, stats, apply passes)
                    roofline["step_traffic_gb"] = t[key]["step_bytes"]
                roofline["algorithmic_gb"] = ALGO_BYTES_PER_PARAM * local_params / 1e9
        except (OSError, ValueError):
            pass

    e2e = None
    if not args.no_e2e:
        e2e_steps = max(3, args.steps // 2)
        ems, h2d, d2h = time_e2e(opt, params, grads, e2e_steps, 2, world)
        e2e = {"value": n_params * e2e_steps / (ems / 1e3) / 1e9, "unit": "Gparams/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": ems / e2e_steps,
               "api": ("LearnedOptimizer.step_host (pinned host grads in, host params out, "
                       f"{E2E_CHUNKS} tensor groups pipelined)" if world == 1 else
                       "ShardedLearnedOptimizer.step, each rank copying its own slice in and "
                       "out (bytes summed over ranks)")}

    clk.__exit__(None, None, None)
    clocks = clk.summary()

    velo = None
    if not args.no_velo and args.feature_set == "small_fc_lopt":
        del opt
        torch.cuda.empty_cache()
        params, grads = make_model(args.workload, dev, seed=0)
        vopt = build_optimizer(params, "velo", args.mode, world, args.strategy, hp)
        vms, vph, _ = time_device(vopt, params, grads, args.steps, args.warmup, world)
        velo = {"optimizer": "VeLO_CUDA (VELO_MLP features + per-tensor LSTM hypernetwork, "
                             "bank of 4 MLPs)",
                "value": n_params * args.steps / (vms / 1e3) / 1e9, "unit": "Gparams/s",
                "ms_per_step": vms / args.steps,
                "step_ms_p10_p50_p90": vph.pop("_step_quantiles", None),
                "ms_per_step_without_param_exchange": vph.pop("_no_exchange_ms", None),
                "host_ms_per_step": vph.pop("_host_ms", None),
                "phase_ms": {k: statistics.mean(v) for k, v in vph.items()}}

    # context: the same parameters stepped by torch's fused
    # AdamW, the usual hand-designed optimizer, on the same device
    adam = None
    if world == 1 and not args.no_velo:
        params, grads = make_model(args.workload, dev, seed=0)
        for p, g in zip(params, grads):
            p.grad = g
        def timed_ms(o):
            for _ in range(args.warmup):
                o.step()
            torch.cuda.synchronize()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record()
            for _ in range(args.steps):
                o.step()
            a1.record()
            torch.cuda.synchronize()
            return a0.elapsed_time(a1) / args.steps

        aopt = torch.optim.AdamW(params, lr=1e-3, fused=True)
        adam = {"torch_adamw_fused_ms_per_step": timed_ms(aopt)}
        del aopt
        # the hand-designed optimizer whose factored second moments small_fc_lopt's
        # features build on (torch's foreach Adafactor)
        aopt = torch.optim.Adafactor(params, lr=1e-2, foreach=True)
        adam["torch_adafactor_foreach_ms_per_step"] = timed_ms(aopt)
        del aopt
        # the reference's own baselines (optim.py:187-217, same conventions),
        # restated on the device (paper_2506_10315_b200.baselines), per tensor
        from paper_2506_10315_b200 import view_2d
        from paper_2506_10315_b200.baselines import adafactor_step, adam_step

        th2 = [p.detach().view(view_2d(p.shape)) for p in params]
        gr2 = [g.view(view_2d(g.shape)) for g in grads]
        ms_ = [torch.zeros_like(t) for t in th2]
        vs_ = [torch.zeros_like(t) for t in th2]
        rs_ = [torch.zeros(t.shape[0], device=dev) for t in th2]
        cs_ = [torch.zeros(t.shape[1], device=dev) for t in th2]

        class _Fn:
            def __init__(self, f):
                self.step = f

        k_ = [0]

        def adam_all():
            k_[0] += 1
            for t, g, m, v in zip(th2, gr2, ms_, vs_):
                adam_step(t, g, m, v, lr=1e-3, t=k_[0])

        def afac_all():
            for t, g, r, c in zip(th2, gr2, rs_, cs_):
                adafactor_step(t, g, r, c, lr=1e-3)

        adam["reference_adam_step_ms_per_step"] = timed_ms(_Fn(adam_all))
        adam["reference_adafactor_step_ms_per_step"] = timed_ms(_Fn(afac_all))
        adam["reference_baselines"] = ("lopt_adam_step / lopt_adafactor_step: the reference's "
                                       "adam_step / adafactor_step (optim.py:187-217) on the "
                                       "device, one call per tensor")
        del params, grads, th2, gr2, ms_, vs_, rs_, cs_

    # config 5 (BASELINE.json): GPT-2 medium, VeLO, cosine schedule + weight
    # decay 0.01, measured in the same run (single GPU; the config's 8-GPU
    # sharding is the --gpus path)
    cfg5 = None
    if world == 1 and not args.no_velo and args.workload == "vit_b16":
        gp, gg = make_model("gpt2_medium", dev, seed=0)
        go = build_optimizer(gp, "velo", args.mode, 1, "range", workload_hparams("gpt2_medium"))
        gms, gph, gl = time_device(go, gp, gg, 10, args.warmup, 1)
        n5 = sum(p.numel() for p in gp)
        cfg5 = {"workload": "gpt2_medium", "optimizer": "VeLO_CUDA", "params": n5,
                "hparams": {k: (repr(v) if k == "schedule" else v)
                            for k, v in workload_hparams("gpt2_medium").items()},
                "ms_per_step": gms / 10, "value": n5 / (gms / 10 / 1e3) / 1e9,
                "unit": "Gparams/s", "kernels_per_step": gl,
                "phase_ms": {k: statistics.mean(v) for k, v in gph.items() if not k.startswith("_")}}
        del go, gp, gg
        torch.cuda.empty_cache()

    # configs 1/2 (BASELINE.json): the 2-layer MNIST MLP, launch-bound -- one
    # captured-graph launch per step
    small = None
    if world == 1 and not args.no_velo and args.workload == "vit_b16":
        small = {}
        for fs in ("small_fc_lopt", "velo"):
            sp, sg = make_model("mnist_mlp", dev, seed=0)
            so = build_optimizer(sp, fs, args.mode, 1, "range", {})
            sms, sph, sl = time_device(so, sp, sg, 200, 10, 1)
            small[fs] = {"ms_per_step": sms / 200, "host_ms_per_step": sph.get("_host_ms"),
                         "params": 101770, "value": 101770 / (sms / 200 / 1e3) / 1e9,
                         "unit": "Gparams/s", "kernels_per_step": sl,
                         "graph_launches_per_step": 1 if so.use_graph else 0}
            del so, sp, sg

    cpu = None
    if not args.no_cpu and world == 1:
        # bounded: three timed steps (plus one warm-up) of the CPU reference
        cpu = cpu_reference(args, n_params, 3, 1, time_budget_s=30.0)[2]

    if rank == 0:
        line = {
            "metric": metric_name(args), "value": value, "unit": "Gparams/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True,
            "step_ms_p10_p50_p90": quant,
            "ms_per_step_without_param_exchange": no_exchange_ms,
            "host_ms_per_step": host_ms,
            "scaling": "strong" if world > 1 else "none", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "mode": args.mode, "param_exchange": gather_used if world > 1 else None,
            "param_exchange_fallback": gather_fallback,
            "config": bench_config(args, hp, n_tensors, n_params, world),
            "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "velo": velo,
            "context": adam, "mnist_mlp": small, "gpt2_medium_velo": cfg5,
            "clocks": clocks, "gpu_launches": launches * args.steps,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
