"""Soak run: many consecutive steps of every optimizer path on ViT-B/16
shapes with fresh synthetic gradients, checking after every step (check_errors)
that nothing fails and the parameters stay finite.

    python tools/soak.py [steps]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_10315_b200 import LearnedOptimizer, VeLO_CUDA  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
dev = torch.device("cuda")
for name, make, n in (("fast small_fc_lopt", lambda ps: LearnedOptimizer(ps, mode="fast"), steps),
                      ("fast VeLO", lambda ps: VeLO_CUDA(ps, mode="fast"), steps // 2),
                      ("strict small_fc_lopt", lambda ps: LearnedOptimizer(ps, mode="strict"),
                       steps // 10)):
    params, grads = bench.make_model("vit_b16", dev, seed=1)
    opt = make(params)
    gen = torch.Generator(device=dev).manual_seed(7)
    t0 = time.perf_counter()
    for k in range(n):
        for p, g in zip(params, grads):
            p.grad = torch.randn(g.shape, device=dev, generator=gen) * 1e-3
        opt.step(loss=2.0) if isinstance(opt, VeLO_CUDA) else opt.step()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    finite = all(bool(torch.isfinite(p).all()) for p in params)
    print(f"{name}: {n} steps in {dt:.1f} s (incl. gradient generation), params finite: {finite}")
    assert finite
    del opt, params, grads
    torch.cuda.empty_cache()
print("soak ok")
