"""One fast-mode step on small shape sets vs the oracle; per-tensor errors."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2506_10315_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402

for shapes in ([(128, 784), (128,), (10, 128), (10,)], [(256, 256)], [(100, 3)], [(3, 1000)]):
    rng = np.random.default_rng(5)
    init = [np.asarray(rng.standard_normal(s) * 0.02, dtype=np.float32) for s in shapes]
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, feature_set="small_fc_lopt", mode="fast")
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [O.OState.zeros(*p.shape) for p in o_params]
    w = O.random_weights(39, seed=0)
    grads = [(rng.standard_normal(p.shape) * 1e-3).astype(np.float32) for p in o_params]
    for p, g in zip(params, grads):
        p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
    opt.step()
    O.opt_step(o_params, o_states, grads, w, O.SMALL_FC_LOPT, 1.0, threads=8)
    for k, (p, q) in enumerate(zip(params, o_params)):
        got = p.detach().cpu().numpy().reshape(-1)
        want = q.reshape(-1)
        err = np.abs(got - want) / (1 + np.abs(want))
        bad = np.nonzero(err > 1e-5)[0]
        print(shapes[k], f"max err {err.max():.2e}", "bad idx:", bad[:8], len(bad))
