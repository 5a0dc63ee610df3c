"""Graph step vs kernel-by-kernel step (same plan, ViT-B/16): per-step GPU
time of each path, alternated, to separate a path effect from clock drift."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from bench import make_model  # noqa: E402
from paper_2506_10315_b200 import LearnedOptimizer  # noqa: E402

params, grads = make_model("vit_b16", "cuda")
for p, g in zip(params, grads):
    p.grad = g
opt = LearnedOptimizer(params, lr=1.0, check_errors=False)


def run(use_graph, n=20, timed=False):
    opt.use_graph = use_graph
    opt.phase_events = [] if timed else None
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(n):
        opt.step()
    b.record()
    torch.cuda.synchronize()
    ph = {}
    if timed:
        for name, x, y in opt.phase_events:
            ph.setdefault(name, []).append(x.elapsed_time(y))
        ph = {k: round(float(np.mean(v)), 4) for k, v in ph.items()}
    opt.phase_events = None
    return a.elapsed_time(b) / n, ph


for _ in range(3):
    run(True, 5)
    run(False, 5)
for rep in range(3):
    for mode in ("graph", "eager", "eager_timed"):
        ms, ph = run(mode == "graph", 20, mode == "eager_timed")
        print(rep, mode, round(ms, 4), ph)
