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


@pytest.mark.parametrize("velo", [False, True])
def test_phase_timed_graph_step_equals_plain_step(velo):
    """The benchmark's phase-timed step (lopt_set_phase_events: event-record
    nodes inside the captured graph, re-pointed every launch) updates exactly
    like the plain kernel-by-kernel step, and its phase windows are positive."""
    import torch

    import paper_2506_10315_b200 as P

    rng, runs = _pair(P, "fast", "velo_mlp" if velo else "small_fc_lopt", velo)
    names_want = ["factors", "stats", "hypernet", "apply"] if velo else ["factors", "stats", "apply"]
    for k in range(5):
        gs = [np.asarray(rng.standard_normal(s) * 1e-2, F32) for s in SHAPES]
        for j, (ps, opt) in enumerate(runs):
            for p, g in zip(ps, gs):
                p.grad = torch.from_numpy(g).cuda()
            timed = j == 0 and k != 3   # graph run; one plain step in between
            opt.phase_events = [] if timed else None
            if velo:
                opt.step(loss=1.5 - 0.1 * k)
            else:
                opt.step()
            if timed:
                torch.cuda.synchronize()
                assert [n for n, _, _ in opt.phase_events] == names_want
                assert all(a.elapsed_time(b) >= 0.0 for _, a, b in opt.phase_events)
                assert sum(a.elapsed_time(b) for _, a, b in opt.phase_events) > 0.0
                opt.phase_events = None
    for a, b in zip(runs[0][0], runs[1][0]):
        assert torch.equal(a.detach(), b.detach())


def test_new_weights_reach_the_launch_parameter_layer3():
    """A single-weight-set fast plan takes layer 3 from the launch parameter
    (DevicePlan::w3c): replacing the weights between steps (lopt_set_weights,
    host or device source) must reach it -- the fast step tracks the strict
    step (which reads the weights from device memory) after the switch."""
    import torch

    import paper_2506_10315_b200 as P

    rng = np.random.default_rng(21)
    init = [np.asarray(rng.standard_normal(s) * 0.05, F32) for s in SHAPES]
    wa = P.random_weights(39, seed=1)
    wb = P.random_weights(39, seed=2, scale=0.35)
    runs = []
    for mode in ("fast", "strict"):
        ps = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
        runs.append((ps, P.LearnedOptimizer(ps, mode=mode, weights=wa)))
    for k in range(4):
        gs = [np.asarray(rng.standard_normal(s) * 1e-2, F32) for s in SHAPES]
        for ps, opt in runs:
            for p, g in zip(ps, gs):
                p.grad = torch.from_numpy(g).cuda()
            if k == 2:
                for plan in opt.plans():
                    if opt.mode == "fast":
                        # device-resident source: the plan reads w3 back
                        dev = torch.from_numpy(wb.packed()).cuda()
                        P._lib.check(plan.L.lopt_set_weights(plan.h, 0, dev.data_ptr(), 1, 0))
                        torch.cuda.synchronize()
                    else:
                        plan.set_weights(0, wb)
            opt.step()
    torch.cuda.synchronize()
    for a, b in zip(runs[0][0], runs[1][0]):
        x, y = a.detach().cpu().numpy(), b.detach().cpu().numpy()
        assert np.max(np.abs(x - y) / (1.0 + np.abs(y))) < 1e-5
