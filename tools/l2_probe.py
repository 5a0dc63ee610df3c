"""Apply-pass time per element with the step's inputs L2-resident (a model
whose 24 B/param working set fits the 126 MB L2) vs the ViT-B/16 step (DRAM):
run under `ncu --cache-control none --metrics gpu__time_duration.sum -k
regex:apply_pair` so consecutive kernels see the L2 the stats pass left.

    python tools/l2_probe.py small|vit
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2506_10315_b200 import LearnedOptimizer

which = sys.argv[1] if len(sys.argv) > 1 else "small"
if which == "vit":
    params, grads = bench.make_model("vit_b16", "cuda")
else:
    g = torch.Generator().manual_seed(0)
    params = [torch.nn.Parameter((torch.randn(768, 768, generator=g) * 0.02).cuda()) for _ in range(4)]
    grads = [(torch.randn(768, 768, generator=g) * 1e-3).cuda() for _ in range(4)]
for p, gr in zip(params, grads):
    p.grad = gr
opt = LearnedOptimizer(params, mode="fast", check_errors=False)
opt.use_graph = False
for _ in range(6):
    opt.step()
torch.cuda.synchronize()
print(which, sum(p.numel() for p in params), "params")
