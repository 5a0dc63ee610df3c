"""Per-CTA balance of the apply kernel: busy time, tensor switches, flat pairs
and unaligned pairs of each CTA's range (a build with -DLOPT_CTA_CLOCK, loaded
through LOPT_SO).

    bash tools/build_variant.sh /tmp/cc.so -DLOPT_CTA_CLOCK
    LOPT_SO=/tmp/cc.so python tools/cta_balance.py [workload]
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2506_10315_b200 import LearnedOptimizer, _lib  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "vit_b16"
params, grads = bench.make_model(wl, torch.device("cuda"))
for p, g in zip(params, grads):
    p.grad = g
opt = LearnedOptimizer(params, feature_set="small_fc_lopt", mode="fast", check_errors=False)
opt.use_graph = False
for _ in range(4):
    opt.step()
torch.cuda.synchronize()
L = _lib.lib()
buf = (ctypes.c_longlong * (64 * 12))()
L.lopt_debug_apply_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32]
assert L.lopt_debug_apply_trace(ctypes.addressof(buf), 64 * 12) == 0
ncta = torch.cuda.get_device_properties(0).multi_processor_count
t = np.array(buf[:5 * ncta], dtype=np.int64).reshape(ncta, 5)
t0 = t[:, 0].min()
start, end = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
busy = end - start
print(f"ctas {ncta}: start max {start.max():.1f} us, end min/avg/max {end.min():.1f} / "
      f"{end.mean():.1f} / {end.max():.1f} us; busy avg {busy.mean():.1f} max {busy.max():.1f} "
      f"(max/avg {busy.max() / busy.mean():.3f})")
order = np.argsort(-busy)
print("slowest CTAs: cta busy_us switches flat_pairs unaligned_pairs")
for b in order[:12]:
    print(f"  {b:4d} {busy[b]:8.1f} {t[b, 2]:4d} {t[b, 3]:6d} {t[b, 4]:6d}")
print("fastest CTAs:")
for b in order[-6:]:
    print(f"  {b:4d} {busy[b]:8.1f} {t[b, 2]:4d} {t[b, 3]:6d} {t[b, 4]:6d}")
sw, fl, un = t[:, 2].astype(float), t[:, 3].astype(float), t[:, 4].astype(float)
X = np.stack([np.ones(ncta), sw, fl, un], 1)
coef, *_ = np.linalg.lstsq(X, busy, rcond=None)
print("busy ~ %.1f + %.2f*switch + %.4f*flat + %.4f*unaligned (us)" % tuple(coef))
print("end-time histogram (us):", np.histogram(end, bins=8)[0].tolist(),
      np.round(np.histogram(end, bins=8)[1], 1).tolist())
