"""Latency/throughput probe of tcgen05.mma kind::f16 at M=128 (one CTA, one
issuing thread): SM cycles per commit round trip for batch sizes, N, and the
A operand in tensor memory vs shared memory."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_10315_b200 import _lib

L = _lib.require_cuda()
out = torch.zeros(1, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for a_smem in (0, 1):
    for N in (32, 64, 128, 256):
        for batch in (1, 13, 64):
            flags = batch | (N << 16) | (a_smem << 28)
            _lib.check(L.lopt_probe_umma(flags, 1000, out.data_ptr(), s))
            torch.cuda.synchronize()
            c = int(out.item())
            print(f"A={'smem' if a_smem else 'tmem'} N={N:3d} batch={batch:3d}: "
                  f"{c:6d} cycles/round {c / batch:7.1f} cycles/MMA")
