"""In-process A/B of apply-kernel configurations on the ViT-B/16 step.

    python tools/apply_ab.py "LOPT_APPLY_VARIANT=3" "LOPT_APPLY_VARIANT=3,LOPT_APPLY_DEBUG=1" ...

Each argument is a comma-separated env assignment list (read by the library
at every launch).  Configurations are interleaved over several rounds on the
same process and inputs; prints the median apply-phase and step time of each.
"""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2506_10315_b200 import LearnedOptimizer

cfgs = [dict(kv.split("=", 1) for kv in a.split(",") if kv) for a in sys.argv[1:]] or [{}]
fs = os.environ.get("AB_FEATURE_SET", "small_fc_lopt")
params, grads = bench.make_model(os.environ.get("AB_WORKLOAD", "vit_b16"), "cuda")
for p, g in zip(params, grads):
    p.grad = g
opt = LearnedOptimizer(params, feature_set=fs, mode="fast", check_errors=False)
keys = sorted({k for c in cfgs for k in c})
res = {i: {"apply": [], "step": []} for i in range(len(cfgs))}
for rnd in range(int(os.environ.get("AB_ROUNDS", "6"))):
    for i, c in enumerate(cfgs):
        for k in keys:
            os.environ.pop(k, None)
        os.environ.update(c)
        for _ in range(3):
            opt.step()
        torch.cuda.synchronize()
        # whole steps (one C call each, as the bench times them)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            opt.step()
        b.record()
        torch.cuda.synchronize()
        res[i]["step"].append(a.elapsed_time(b) / 10)
        # phases (separate calls: includes host gaps, for reference only)
        opt.phase_events = []
        for _ in range(3):
            opt.step()
        torch.cuda.synchronize()
        res[i]["apply"] += [x.elapsed_time(y) for n, x, y in opt.phase_events if n == "apply"]
        opt.phase_events = None
for i, c in enumerate(cfgs):
    print(f"{c}: apply median {statistics.median(res[i]['apply']):.4f} ms "
          f"(min {min(res[i]['apply']):.4f}), step median {statistics.median(res[i]['step']):.4f} ms")
