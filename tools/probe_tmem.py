"""TMEM throughput probe: bytes per SM cycle of tcgen05.ld / tcgen05.st with
4..32 warps of one CTA (one SM)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2506_10315_b200 import _lib

L = _lib.require_cuda()
out = torch.zeros(64, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
names = {0: "ld x16", 1: "ld x32", 2: "st x16"}
cols = {0: 16, 1: 32, 2: 16}
for mode in (0, 1, 2):
    for warps in (4, 8, 16, 32):
        per, rounds = 8, 200
        out.zero_()
        _lib.check(L.lopt_probe_tmem(warps, mode, per, rounds, out.data_ptr(), s))
        torch.cuda.synchronize()
        cyc = max(int(v) for v in out[:warps].tolist())
        byts = warps * rounds * per * 32 * cols[mode] * 4
        print(f"{names[mode]} warps={warps:2d}: {cyc / (rounds * per):8.1f} cycles per op per warp, "
              f"{byts / cyc:7.1f} B/cycle/SM")
