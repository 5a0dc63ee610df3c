"""ViT-B/16 fast step with N stand-in peer arenas on the same GPU (the fused
all-gather's stores, bulk or element-wise): step time, and under ncu the apply
kernel's instruction count with and without peers.

    python tools/peer_probe.py N [steps]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import bench
from paper_2506_10315_b200 import LearnedOptimizer

n_peers = int(sys.argv[1]) if len(sys.argv) > 1 else 7
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
params, grads = bench.make_model("vit_b16", "cuda")
total = sum(p.numel() for p in params)
arena = torch.empty(total, device="cuda")
off, ps = 0, []
for p in params:
    n = p.numel()
    arena[off:off + n].copy_(p.detach().reshape(-1))
    ps.append(torch.nn.Parameter(arena[off:off + n].view(p.shape)))
    off += n
for p, g in zip(ps, grads):
    p.grad = g
peers = [torch.empty(total, device="cuda") for _ in range(n_peers)]
opt = LearnedOptimizer(ps, mode="fast", check_errors=False)
if peers:
    opt.set_peer_copies([q.data_ptr() - arena.data_ptr() for q in peers])
for _ in range(3):
    opt.step()
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(steps):
    opt.step()
b.record()
torch.cuda.synchronize()
print(f"peers={n_peers} bulk={os.environ.get('LOPT_PEER_SCALAR') is None}: "
      f"{a.elapsed_time(b) / steps:.3f} ms/step")
if peers:
    assert all(torch.equal(q, arena) for q in peers)
