import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2506_10315_b200 as P
from oracle import oracle as O
shapes = [(128, 784), (128,), (10, 128), (10,)]
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
got = params[2].detach().cpu().numpy()
print("row0 unchanged:", np.count_nonzero(got[0] == init[2][0]), "/128")
print("row0 got-want:", (got[0] - o_params[2][0])[:6])
print("row0 delta want:", (o_params[2][0] - init[2][0])[:6])
print("row0 delta got:", (got[0] - init[2][0])[:6])
print("row1 got-want:", np.abs(got[1] - o_params[2][1]).max())
q = opt.state[params[2]]["quad"].cpu().numpy()
print("state M1 row0 ok:", np.abs(q[:128, 0] - o_states[2].M[0][0]).max())
