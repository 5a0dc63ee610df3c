"""Pipeline trace of the apply kernel (CTA 0, first 64 tiles): clock64 at
producer stage (0), A data ready (1), A operands done (2), MMA1 go (3),
B acc1 ready (4), MMA2 go (5), C acc2 ready (6).

    LOPT_APPLY_DEBUG=32 python tools/trace_apply.py
"""
import ctypes
import os
import sys

import numpy as np

os.environ.setdefault("LOPT_APPLY_DEBUG", "32")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_10315_b200 import LearnedOptimizer, _lib  # noqa: E402

params, grads = bench.make_model("vit_b16", torch.device("cuda"))
for p, g in zip(params, grads):
    p.grad = g
opt = LearnedOptimizer(params, feature_set="small_fc_lopt", mode="fast", check_errors=False)
for _ in range(3):
    opt.step()
torch.cuda.synchronize()
L = _lib.lib()
buf = (ctypes.c_longlong * (64 * 12))()
L.lopt_debug_apply_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
assert L.lopt_debug_apply_trace(ctypes.addressof(buf), 64 * 12) == 0
t = np.array(buf[:], dtype=np.int64).reshape(64, 12)
# the first warp of each role's warpgroup 0 records: even tiles; columns in
# pipeline order: prod, A data ready, A features done (before the TMEM slot
# wait), A operands stored, MMA1, B loop top, B acc1 ready, MMA2, C before
# acc2 wait, C acc2 ready, C done
ev = t[0::2][:, [0, 1, 8, 2, 3, 10, 4, 5, 9, 6, 7]]
ev = ev - ev[0, 0]
names = ["prod", "A_in", "A_feat", "A_out", "mma1", "B_top", "B_in", "mma2", "C_top", "C_in",
         "C_end"]
print("tile " + " ".join(f"{n:>8s}" for n in names))
for k in range(ev.shape[0]):
    print(f"{2 * k:4d} " + " ".join(f"{v:8d}" for v in ev[k]))
s_ = ev[4:]
print("cycles per tile (even-tile spacing / 2):",
      " ".join(f"{n}={v:.0f}" for n, v in zip(names, np.diff(s_, axis=0).mean(axis=0) / 2)))
lat = (s_[:, 1:] - s_[:, :-1]).mean(axis=0)
print("mean stage latency:", " ".join(f"{names[k]}->{names[k+1]}={v:.0f}" for k, v in enumerate(lat)))
