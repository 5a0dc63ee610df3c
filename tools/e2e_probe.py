"""PCIe bandwidths and step_host chunk counts on ViT-B/16."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
from paper_2506_10315_b200 import LearnedOptimizer

N = 86567656
h = torch.empty(N, dtype=torch.float32).pin_memory()
d = torch.empty(N, dtype=torch.float32, device="cuda")
for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
    fn(); torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): fn()
    b.record(); torch.cuda.synchronize()
    print(name, f"{N*4*5/(a.elapsed_time(b)/1e3)/1e9:.1f} GB/s")
h2 = torch.empty(N, dtype=torch.float32).pin_memory()
d2 = torch.empty(N, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(5):
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
print("bidirectional", f"{2*N*4*5/(time.perf_counter()-t0)/1e9:.1f} GB/s total")
params, grads = bench.make_model("vit_b16", torch.device("cuda"))
opt = LearnedOptimizer(params, mode="fast", check_errors=False)
hg = [g.cpu().pin_memory() for g in grads]
hp = [torch.empty(p.shape).pin_memory() for p in params]
for ch in (4, 8, 16, 32):
    opt._host_step = None
    for _ in range(3): opt.step_host(hg, hp, chunks=ch)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): opt.step_host(hg, hp, chunks=ch)
    b.record(); torch.cuda.synchronize()
    print("chunks", ch, f"{a.elapsed_time(b)/5:.2f} ms")
# host enqueue cost of one step_host call (the GPU may wait on the CPU)
for ch in (8, 32):
    opt._host_step = None
    for _ in range(3): opt.step_host(hg, hp, chunks=ch)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(5): opt.step_host(hg, hp, chunks=ch)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print("chunks", ch, f"enqueue {(t1 - t0) / 5 * 1e3:.2f} ms/step, wall {(t2 - t0) / 5 * 1e3:.2f} ms/step")
