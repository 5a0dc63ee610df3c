"""Co-residency probe: can the stats pass of one tensor group run on the SMs
beside the apply pass of another (the apply kernel is issue/latency-bound at
~27 % of HBM; the stats pass is HBM-bound)?  ViT-B/16 split into two groups of
equal size; times apply(A) alone, stats(B) alone, and both launched together
on two streams.  Run with LOPT_SO pointing at a build whose apply kernel
leaves registers for a stats CTA (tools/build_variant.sh ... -DLOPT_APPLY_MAXNREG=112
-DLOPT_STAT_THREADS=128 -DLOPT_STAT_MINB=8)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
from bench import make_model  # noqa: E402
from paper_2506_10315_b200 import LearnedOptimizer  # noqa: E402


def timed(fn, reps=20):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    params, grads = make_model(os.environ.get("WL", "vit_b16"), "cuda")
    for p, g in zip(params, grads):
        p.grad = g
    order = sorted(range(len(params)), key=lambda k: -params[k].numel())
    A, B, sa, sb = [], [], 0, 0
    for k in order:
        if sa <= sb:
            A.append(params[k]); sa += params[k].numel()
        else:
            B.append(params[k]); sb += params[k].numel()
    opt = LearnedOptimizer([{"params": A}, {"params": B}], lr=1.0)
    opt.use_graph = False
    opt.step()
    torch.cuda.synchronize()
    pa, pb = opt._plans[0][1], opt._plans[1][1]
    for pl in (pa, pb):
        pl.set_step(1.0, 0.0, 5)
        pl.factor_partials()
        pl.factor_finalize()
        pl.feature_stats()
    torch.cuda.synchronize()
    s2 = torch.cuda.Stream()
    main_s = torch.cuda.current_stream()

    def both(with_factor):
        e0 = torch.cuda.Event()
        e0.record(main_s)
        pa.apply()   # launched first: one CTA per SM, the stats CTAs fill the rest
        s2.wait_event(e0)
        with torch.cuda.stream(s2):
            if with_factor:
                pb.factor_partials()
                pb.factor_finalize()
            pb.feature_stats()
        e1 = torch.cuda.Event()
        e1.record(s2)
        main_s.wait_event(e1)

    def statsb_factor():
        pb.factor_partials()
        pb.factor_finalize()
        pb.feature_stats()

    r = {
        "params_A": sa, "params_B": sb,
        "apply_A_ms": timed(pa.apply),
        "stats_B_ms": timed(pb.feature_stats),
        "factor_stats_B_ms": timed(statsb_factor),
        "both_ms": timed(lambda: both(False)),
        "both_with_factor_ms": timed(lambda: both(True)),
    }
    r["serial_ms"] = r["apply_A_ms"] + r["stats_B_ms"]
    r["hidden_frac"] = (r["serial_ms"] - r["both_ms"]) / r["stats_B_ms"]
    print(r)


if __name__ == "__main__":
    main()
