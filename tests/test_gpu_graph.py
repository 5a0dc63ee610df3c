"""The captured-graph step (lopt_graph_step): the whole step -- scalars,
factor pass, stats pass, VeLO hypernetwork, apply pass -- replayed from one
CUDA graph per plan must give exactly what the kernel-by-kernel step gives,
across changing lr / weight decay / step counters, re-pointed gradients and
both modes; and it must cut the launches per step to one graph launch."""

import numpy as np
import pytest

from conftest import F32

pytestmark = pytest.mark.gpu

SHAPES = [(256, 192), (256,), (96, 256), (33, 70), (1, 130), (7,)]


def _pair(P, mode, fs, velo=False):
    import torch

    rng = np.random.default_rng(4)
    init = [np.asarray(rng.standard_normal(s) * 0.05, F32) for s in SHAPES]
    out = []
    for use_graph in (True, False):
        ps = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
        if velo:
            opt = P.VeLO_CUDA(ps, mode=mode, weight_decay=0.01,
                              hypernet=P.VeLOHyperNet(seed=1))
        else:
            opt = P.LearnedOptimizer(ps, feature_set=fs, mode=mode, weight_decay=0.01,
                                     schedule=P.ScheduleConfig("cosine", 0.9, 0.05, 2, 12))
        opt.use_graph = use_graph
        out.append((ps, opt))
    return rng, out


@pytest.mark.parametrize("mode,fs,velo", [("fast", "small_fc_lopt", False),
                                          ("fast", "velo_mlp", False),
                                          ("strict", "small_fc_lopt", False),
                                          ("fast", "velo_mlp", True),
                                          ("strict", "velo_mlp", True)])
def test_graph_step_equals_kernel_by_kernel_step(mode, fs, velo):
    import torch

    import paper_2506_10315_b200 as P

    rng, runs = _pair(P, mode, fs, velo)
    for k in range(8):
        gs = [np.asarray(rng.standard_normal(s) * 1e-2, F32) for s in SHAPES]
        for ps, opt in runs:
            # fresh gradient tensors every other step: the plan re-points
            # them (lopt_rebind_tensors) and the captured graph stays valid
            if k % 2 == 0 or ps[0].grad is None:
                for p, g in zip(ps, gs):
                    p.grad = torch.from_numpy(g).cuda()
            else:
                for p, g in zip(ps, gs):
                    p.grad.copy_(torch.from_numpy(g))
            if velo:
                opt.step(loss=2.0 - 0.1 * k)
            else:
                opt.step()
    (pa, oa), (pb, ob) = runs
    torch.cuda.synchronize()
    for a, b in zip(pa, pb):
        assert torch.equal(a.detach(), b.detach())
        assert torch.equal(oa.state[a]["quad"], ob.state[b]["quad"])
    if velo:
        assert torch.equal(oa._lstm[0][0], ob._lstm[0][0])
    assert oa.plans()[0].gexec_ready()


def test_graph_step_nonfinite_gradient_changes_nothing():
    import torch

    import paper_2506_10315_b200 as P

    a = torch.nn.Parameter(torch.ones(64, 32, device="cuda"))
    opt = P.LearnedOptimizer([a])
    a.grad = torch.full((64, 32), 0.01, device="cuda")
    opt.step()
    snap = a.detach().clone()
    q = opt.state[a]["quad"].clone()
    a.grad[3, 3] = float("nan")
    with pytest.raises(P.OptimError):
        opt.step()
    assert torch.equal(a.detach(), snap) and torch.equal(opt.state[a]["quad"], q)
    a.grad[3, 3] = 0.01
    opt.step()
    assert torch.isfinite(a).all() and not torch.equal(a.detach(), snap)


def test_phase_timed_step_equals_graph_step():
    """The benchmark's phase-timed step (lopt_set_phase_events: one C step
    recording four events) updates exactly like the graph step, and its phase
    windows are positive and add up to the step."""
    import torch

    import paper_2506_10315_b200 as P

    rng, runs = _pair(P, "fast", "small_fc_lopt")
    for k in range(4):
        gs = [np.asarray(rng.standard_normal(s) * 1e-2, F32) for s in SHAPES]
        for j, (ps, opt) in enumerate(runs):
            for p, g in zip(ps, gs):
                p.grad = torch.from_numpy(g).cuda()
            opt.phase_events = [] if j == 1 else None
            opt.step()
            if j == 1:
                torch.cuda.synchronize()
                names = [n for n, _, _ in opt.phase_events]
                assert names == ["factors", "stats", "apply"]
                assert all(a.elapsed_time(b) > 0.0 for _, a, b in opt.phase_events)
                opt.phase_events = None
    for a, b in zip(runs[0][0], runs[1][0]):
        assert torch.equal(a.detach(), b.detach())
