"""Latency/throughput probe of tcgen05.mma kind::f16 at M=128 (one CTA):
SM cycles per commit round trip for batch sizes and N, A in tensor memory vs
shared memory, and with 1-4 warps issuing independent MMA streams."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_10315_b200 import _lib

L = _lib.require_cuda()
out = torch.zeros(4, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for a_smem in (0, 1):
    for N in (32, 64, 128, 256):
        for batch in (1, 13, 64):
            flags = batch | (N << 16) | (a_smem << 28)
            _lib.check(L.lopt_probe_umma(flags, 1000, out.data_ptr(), s))
            torch.cuda.synchronize()
            c = int(out[0].item())
            print(f"A={'smem' if a_smem else 'tmem'} N={N:3d} batch={batch:3d}: "
                  f"{c:6d} cycles/round {c / batch:7.1f} cycles/MMA")
for N in (32, 64, 128):
    for batch in (16, 64):
        flags = batch | (N << 16) | (1 << 29)
        _lib.check(L.lopt_probe_umma(flags, 1000, out.data_ptr(), s))
        torch.cuda.synchronize()
        c = int(out[0].item())
        print(f"A=tmem N={N:3d} batch={batch:3d} 4 independent accumulators: "
              f"{c / batch:7.1f} cycles/MMA")
for a_smem in (0, 1):
    for N in (32, 64):
        for issuers in (2, 3, 4):
            for batch in (10, 64):
                out.zero_()
                flags = batch | (issuers << 12) | (N << 16) | (a_smem << 28)
                _lib.check(L.lopt_probe_umma(flags, 500, out.data_ptr(), s))
                torch.cuda.synchronize()
                c = [int(v) for v in out.tolist()[:issuers]]
                mx = max(c)
                print(f"A={'smem' if a_smem else 'tmem'} issuers={issuers} N={N} batch={batch:3d}: "
                      f"max {mx} cycles/round per issuer, aggregate {mx / (batch * issuers):6.1f} cycles/MMA")
for a_smem in (0, 1):
    for N in (32, 64, 128, 256):
        for issuers in (1, 2, 4):
            for batch in (10, 64):
                out.zero_()
                flags = batch | (issuers << 12) | (N << 16) | (a_smem << 28) | (1 << 30)
                _lib.check(L.lopt_probe_umma(flags, 500, out.data_ptr(), s))
                torch.cuda.synchronize()
                c = [int(v) for v in out.tolist()[:issuers]]
                mx = max(c)
                print(f"WARP-WIDE A={'smem' if a_smem else 'tmem'} issuers={issuers} N={N} batch={batch:3d}: "
                      f"max {mx} cycles/round, aggregate {mx / (batch * issuers):6.1f} cycles/MMA")
