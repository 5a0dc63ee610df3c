"""GPU parity of the strict (bitwise) CUDA path against the oracle and the
reference-generated golden fixtures.  Needs a B200: run with -m gpu."""

import numpy as np
import pytest

from conftest import F32, advanced_state, load_golden

pytestmark = pytest.mark.gpu

ENGINE_SHAPES = [(1, 1), (1, 130), (130, 1), (5, 64), (7, 63), (3, 65), (33, 70), (64, 64),
                 (17, 129)]
MODEL_SHAPES = [(16, 98), (16, 1), (10, 16), (10, 1)]


@pytest.fixture(scope="module")
def P():
    import torch

    assert torch.cuda.is_available()
    import paper_2506_10315_b200 as P

    return P


def _dev_state(P, O, s):
    return P.DeviceOptState.from_arrays(s.M, s.V, s.r, s.c, s.t)


def _golden_state(O, G, key, m, n):
    s = O.OState.zeros(m, n)
    for i in range(3):
        s.M[i] = G[f"{key}/M{i}"]
        s.r[i] = G[f"{key}/r{i}"]
        s.c[i] = G[f"{key}/c{i}"]
    s.V = G[f"{key}/V"]
    s.t = int(G[f"{key}/t"][0])
    return s


@pytest.mark.parametrize("spec_name", ["small_fc_lopt", "velo_mlp"])
@pytest.mark.parametrize("shape", ENGINE_SHAPES)
def test_step_fused_strict_bitwise_vs_reference(P, oracle, spec_name, shape):
    """engine.step_fused on the device == reference step_fused, bit for bit
    (same advanced state; the device f64 sums use another order, which the
    f32 scale does not see on these instances)."""
    import torch

    O = oracle
    G = load_golden("engine_cases.npz")
    m, n = shape
    key = f"{spec_name}/{m}x{n}"
    s = _golden_state(O, G, key, m, n)
    spec = P.spec_by_name(spec_name)
    W = torch.from_numpy(G[key + "/W"]).cuda()
    g = torch.from_numpy(G[key + "/g"]).cuda()
    w = P.random_weights(spec.d_feat, seed=int(G[key + "/wseed"][0]))
    sumsq, count = P.fused_stats(W, g, _dev_state(P, O, s), spec)
    np.testing.assert_allclose(sumsq.cpu().numpy(), G[key + "/sumsq_w1"], rtol=1e-12)
    for lr in (1.0, 0.3):
        out, rep = P.step_fused(W, g, _dev_state(P, O, s), w, spec, lr=lr)
        want = G[key + f"/out_lr{lr}"]
        got = out.cpu().numpy()
        assert got.tobytes() == want.tobytes(), np.argwhere(got != want)[:5]
        assert rep["max_abs_update"] == pytest.approx(float(G[key + f"/maxabs_lr{lr}"][0]),
                                                      rel=0, abs=0)


def test_zero_network_step_is_bitwise_noop(P, oracle):
    """test_engine.py:249-259 / acceptance 3 on the device."""
    import torch

    rng = np.random.default_rng(1)
    m, n = 33, 70
    s, g = advanced_state(rng, m, n, steps=2)
    W = rng.standard_normal((m, n)).astype(F32)
    W[0, 0] = -0.0
    W[0, 1] = 0.0
    out, _ = P.step_fused(torch.from_numpy(W).cuda(), torch.from_numpy(g).cuda(),
                          _dev_state(P, oracle, s), P.zero_weights(39), P.small_fc_lopt_spec())
    assert out.cpu().numpy().tobytes() == W.tobytes()


def test_overflow_raises_typed_error(P, oracle):
    """test_engine.py:380-391."""
    import torch

    rng = np.random.default_rng(0)
    s, g = advanced_state(rng, 6, 6, steps=1)
    W = rng.standard_normal((6, 6)).astype(F32)
    w = P.random_weights(39, seed=0)
    w.layers[-1][1][1] = 1e7
    with pytest.raises(P.UpdateOverflowError):
        P.step_fused(torch.from_numpy(W).cuda(), torch.from_numpy(g).cuda(),
                     _dev_state(P, oracle, s), w, P.small_fc_lopt_spec())


def test_mismatched_weights_rejected(P, oracle):
    import torch

    rng = np.random.default_rng(0)
    s, g = advanced_state(rng, 4, 4, steps=1)
    W = torch.from_numpy(rng.standard_normal((4, 4)).astype(F32)).cuda()
    with pytest.raises(P.EngineError):
        P.step_fused(W, torch.from_numpy(g).cuda(), _dev_state(P, oracle, s),
                     P.random_weights(29, seed=0), P.small_fc_lopt_spec())


# ---------------------------------------------------------------------------
# optimizer facade, multi-step trajectories


def _model(P, init, shapes):
    import torch

    return [torch.nn.Parameter(torch.from_numpy(init[j].reshape(s).copy()).cuda())
            for j, s in enumerate(shapes)]


@pytest.mark.parametrize("run", ["small_const", "velo_cos_wd"])
def test_optimizer_strict_trajectory_bitwise_vs_reference(P, oracle, run):
    import torch

    G = load_golden("optstep_cases.npz")
    cfg = {
        "small_const": dict(fs="small_fc_lopt", sched=P.ScheduleConfig("constant", 1.0), wd=0.0,
                            wseed=0),
        "velo_cos_wd": dict(fs="velo_mlp", sched=P.ScheduleConfig("cosine", 0.8, 0.05, 2, 8),
                            wd=0.01, wseed=1),
    }[run]
    init = [G[f"{run}/init/param{j}"] for j in range(len(MODEL_SHAPES))]
    params = _model(P, init, MODEL_SHAPES)
    d = 39 if cfg["fs"] == "small_fc_lopt" else 29
    opt = P.LearnedOptimizer(params, weight_decay=cfg["wd"], feature_set=cfg["fs"],
                             weights=P.random_weights(d, seed=cfg["wseed"]),
                             schedule=cfg["sched"], mode="strict")
    grng = np.random.default_rng(78)
    for step in range(6):
        for p in params:
            shape2 = P.view_2d(p.shape)
            g = (grng.standard_normal(shape2) * 1e-2).astype(F32)
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step()
        for j, p in enumerate(params):
            want = G[f"{run}/step{step}/param{j}"].reshape(-1)
            got = p.detach().cpu().numpy().reshape(-1)
            assert got.tobytes() == want.tobytes(), (step, j, np.abs(got - want).max())


def test_optimizer_vs_oracle_vit_like_shapes_one_step(P, oracle):
    """ViT-B/16 block shapes (incl. a 768-vector and a 3-D tensor via the view
    rule) after several steps: strict device == oracle bitwise."""
    import torch

    shapes = [(2304, 768), (768,), (3072, 768), (1, 197, 768), (768, 3, 4, 4)]
    rng = np.random.default_rng(3)
    init = [(rng.standard_normal(s) * 0.02).astype(F32) for s in shapes]
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, feature_set="small_fc_lopt", mode="strict")
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [oracle.OState.zeros(*p.shape) for p in o_params]
    w = oracle.random_weights(39, seed=0)
    for step in range(3):
        grads = [(rng.standard_normal(p.shape) * 1e-3).astype(F32) for p in o_params]
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step()
        oracle.opt_step(o_params, o_states, grads, w, oracle.SMALL_FC_LOPT, 1.0, threads=8)
    for p, q in zip(params, o_params):
        got = p.detach().cpu().numpy().reshape(-1)
        want = q.reshape(-1)
        bad = np.count_nonzero(got != want)
        # bitwise: the device's f64 reduction orders differ from numpy's, but
        # on these inputs no f32 rounding of a factor mean, normalization scale
        # or feature flips
        assert bad == 0, (q.shape, bad, np.max(np.abs(got - want)))


def test_nonfinite_gradient_raises_and_changes_nothing(P):
    """optim.py:160-165 / test_optim.py:186-197."""
    import torch

    a = torch.nn.Parameter(torch.ones(2, 2, device="cuda"))
    b = torch.nn.Parameter(torch.ones(3, 3, device="cuda"))
    opt = P.LearnedOptimizer([a, b], mode="strict")
    a.grad = torch.ones(2, 2, device="cuda")
    bad = torch.ones(3, 3, device="cuda")
    bad[0, 0] = float("nan")
    b.grad = bad
    with pytest.raises(P.OptimError, match="param1"):
        opt.step()
    assert torch.equal(a.detach(), torch.ones(2, 2, device="cuda"))
    assert torch.equal(b.detach(), torch.ones(3, 3, device="cuda"))
    for p in (a, b):   # no accumulator was committed either
        st = opt.state[p]
        assert not st["quad"].any() and not st["row_factors"].any() and not st["col_factors"].any()


def test_decay_runs_after_update_exactly(P):
    """test_optim.py:153-163: zero net, lr 1, wd 0.1 -> theta * f32(0.9)."""
    import torch

    rng = np.random.default_rng(5)
    x = rng.standard_normal((4, 4)).astype(F32)
    p = torch.nn.Parameter(torch.from_numpy(x.copy()).cuda())
    opt = P.LearnedOptimizer([p], weight_decay=0.1, weights=P.zero_weights(39), mode="strict")
    p.grad = torch.ones(4, 4, device="cuda")
    opt.step()
    assert p.detach().cpu().numpy().tobytes() == (x * F32(1.0 - 1.0 * 0.1)).tobytes()


def test_warmup_lr_sampled_before_increment(P):
    """test_optim.py:121-133: warmup -> lr 0 on the first step -> no change."""
    import torch

    x = torch.randn(6, 6, device="cuda")
    p = torch.nn.Parameter(x.clone())
    opt = P.LearnedOptimizer([p], schedule=P.ScheduleConfig("cosine", 1.0, 0.0, 2, 4),
                             mode="strict")
    p.grad = torch.randn(6, 6, device="cuda")
    opt.step()
    assert torch.equal(p.detach(), x) and opt.T == 1


def test_state_dict_resume_is_bitwise(P):
    """Acceptance 10 / test_optim.py:307-331 on the device."""
    import torch

    shapes = [(6, 9), (11, 4), (7,)]
    rng = np.random.default_rng(9)
    init = [rng.standard_normal(s).astype(F32) for s in shapes]
    grads = [[rng.standard_normal(s).astype(F32) for s in shapes] for _ in range(4)]
    sched = P.ScheduleConfig("cosine", 0.8, 0.0, 1, 4)

    def run(stop=None, resume=None):
        params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
        opt = P.LearnedOptimizer(params, weight_decay=0.01, schedule=sched, mode="strict")
        start = 0
        if resume is not None:
            for p, v in zip(params, resume[0]):
                p.data.copy_(v)
            opt.load_state_dict(resume[1])
            start = opt.T
        for k in range(start, 4 if stop is None else stop):
            for p, g in zip(params, grads[k]):
                p.grad = torch.from_numpy(g).cuda()
            opt.step()
        return params, opt

    full, _ = run()
    half, opt = run(stop=2)
    ck = ([p.detach().clone() for p in half], opt.state_dict())
    resumed, opt2 = run(resume=ck)
    assert opt2.T == 4
    for a, b in zip(full, resumed):
        assert a.detach().cpu().numpy().tobytes() == b.detach().cpu().numpy().tobytes()


def test_hundred_steps_relative_l2_vs_oracle(P, oracle):
    """North-star tolerance check: params and states after 100 steps on the
    MNIST-shaped MLP, strict mode, relative L2 vs the oracle."""
    import torch

    shapes = [(128, 784), (128,), (10, 128), (10,)]
    rng = np.random.default_rng(11)
    init = [(rng.standard_normal(s) * 0.05).astype(F32) for s in shapes]
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, feature_set="velo_mlp", weight_decay=0.01, mode="strict",
                             schedule=P.ScheduleConfig("cosine", 0.5, 0.01, 5, 100))
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [oracle.OState.zeros(*p.shape) for p in o_params]
    w = oracle.random_weights(29, seed=0)
    for step in range(100):
        grads = [(rng.standard_normal(p.shape) * 1e-2).astype(F32) for p in o_params]
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step()
        lr = oracle.schedule_lr("cosine", 0.5, 0.01, 5, 100, step)
        oracle.opt_step(o_params, o_states, grads, w, oracle.VELO_MLP, lr, weight_decay=0.01)
    for p, q in zip(params, o_params):
        got = p.detach().cpu().numpy().reshape(-1).astype(np.float64)
        want = q.reshape(-1).astype(np.float64)
        rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
        assert rel <= 1e-6, rel
    for p, s in zip(params, o_states):
        quad = opt.state[p]["quad"].cpu().numpy()
        assert quad[:, 3].tobytes() == s.V.reshape(-1).tobytes()
        assert quad[:, 0].tobytes() == s.M[0].reshape(-1).tobytes()


@pytest.mark.parametrize("mode", ["strict", "fast"])
@pytest.mark.parametrize("spec_name", ["small_fc_lopt", "velo_mlp"])
@pytest.mark.parametrize("shape", [(33, 70), (17, 129), (1, 130), (64, 64)])
def test_range_operator_pair_matches_whole_tensor(P, oracle, spec_name, shape, mode):
    """engine.py:619-710 range-level pair as the sharded step uses it
    (distsim.py:489-490,513-514): fused_stats over [0,k) and [k,mn) add up to
    the whole-tensor stats (acceptance 9), and fused_apply over the two ranges
    with the merged stats writes exactly what step_fused does (itself pinned
    bitwise to the reference above) -- bit for bit."""
    import torch

    O = oracle
    G = load_golden("engine_cases.npz")
    m, n = shape
    key = f"{spec_name}/{m}x{n}"
    s = _golden_state(O, G, key, m, n)
    spec = P.spec_by_name(spec_name)
    W = torch.from_numpy(G[key + "/W"]).cuda()
    g = torch.from_numpy(G[key + "/g"]).cuda()
    w = P.random_weights(spec.d_feat, seed=int(G[key + "/wseed"][0]))
    mn = m * n
    k = mn // 3
    whole = P.fused_stats(W, g, _dev_state(P, O, s), spec, mode=mode)
    a = P.fused_stats(W, g, _dev_state(P, O, s), spec, lo=0, hi=k, mode=mode)
    b = P.fused_stats(W, g, _dev_state(P, O, s), spec, lo=k, hi=mn, mode=mode)
    assert a.count + b.count == whole.count == mn
    merged = a.sumsq + b.sumsq
    # strict: f64 sums of exact squares; fast: f32 per-thread partials (the
    # reference's own additivity bound is 1e-6, acceptance 9)
    np.testing.assert_allclose(merged.cpu().numpy(), whole.sumsq.cpu().numpy(),
                               rtol=1e-12 if mode == "strict" else 1e-6)
    ref, _ = P.step_fused(W, g, _dev_state(P, O, s), w, spec, lr=0.3, mode=mode)
    out = torch.full_like(W, float("nan"))
    st = _dev_state(P, O, s)
    mx0 = P.fused_apply(W, g, st, w, spec, (merged, mn), out, lr=0.3, lo=0, hi=k, mode=mode)
    assert torch.isnan(out.view(-1)[k:]).all()
    mx1 = P.fused_apply(W, g, st, w, spec, P.FeatureStats(merged, mn), out, lr=0.3,
                        lo=k, hi=mn, mode=mode)
    if mode == "strict":
        assert out.cpu().numpy().tobytes() == ref.cpu().numpy().tobytes()
    else:   # merged range sums may differ from the whole-tensor sums in the last f64 bits
        a_, r_ = out.cpu().numpy().astype(np.float64), ref.cpu().numpy()
        assert (np.abs(a_ - r_) / (1 + np.abs(r_))).max() <= 1e-7
    assert max(mx0, mx1) > 0
    # a partial-range count normalizes by that count, as the reference does
    # (engine.py:657-710 accepts any FeatureStats): against the oracle
    out2 = torch.full_like(W, float("nan"))
    P.fused_apply(W, g, st, w, spec, a, out2, lr=0.3, lo=0, hi=k, mode=mode)
    want, _ = O.fused_apply(G[key + "/W"], G[key + "/g"], s, O.random_weights(spec.d_feat, seed=int(G[key + "/wseed"][0])),
                            O.KIND_BY_NAME[spec_name], a.sumsq.cpu().numpy(), a.count, lr=0.3, lo=0, hi=k)
    got = out2.cpu().numpy().reshape(-1)[:k]
    want = want.reshape(-1)[:k]
    if mode == "strict":
        assert got.tobytes() == want.tobytes()
    else:
        assert (np.abs(got.astype(np.float64) - want) / (1 + np.abs(want))).max() <= 1e-5


def test_torch_lr_scheduler_drives_group_lr(P):
    """torch.optim.lr_scheduler works through param_groups[i]["lr"]: a
    StepLR-halved run equals a run whose group lr is set by hand."""
    import torch

    shapes = [(32, 48), (32,)]
    rng = np.random.default_rng(9)
    init = [np.asarray(rng.standard_normal(s) * 0.05, dtype=F32) for s in shapes]
    grads = [[np.asarray(rng.standard_normal(s) * 1e-2, dtype=F32) for s in shapes]
             for _ in range(4)]
    a = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    b = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    oa = P.LearnedOptimizer(a, lr=0.8, weight_decay=0.01)
    ob = P.LearnedOptimizer(b, lr=0.8, weight_decay=0.01)
    sched = torch.optim.lr_scheduler.StepLR(oa, step_size=2, gamma=0.5)
    for k, gs in enumerate(grads):
        for p, q, g in zip(a, b, gs):
            p.grad = torch.from_numpy(g).cuda()
            q.grad = torch.from_numpy(g).cuda()
        ob.param_groups[0]["lr"] = 0.8 * (0.5 ** (k // 2))
        oa.step()
        ob.step()
        sched.step()
    for p, q in zip(a, b):
        assert p.detach().cpu().numpy().tobytes() == q.detach().cpu().numpy().tobytes()
    assert oa.param_groups[0]["lr"] == 0.8 * 0.25


def test_functional_opt_step_matches_step(P):
    """opt_step(opt, grads, loss) (optim.py:144-180's functional surface):
    same result as assigning .grad and stepping; count and shape errors."""
    import torch

    rng = np.random.default_rng(5)
    shapes = [(16, 9), (9,)]
    init = [(rng.standard_normal(s) * 0.1).astype(F32) for s in shapes]
    grads = [torch.from_numpy((rng.standard_normal(s) * 1e-2).astype(F32)).cuda() for s in shapes]
    a = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    b = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    oa, ob = P.LearnedOptimizer(a, mode="strict"), P.LearnedOptimizer(b, mode="strict")
    P.opt_step(oa, grads)
    for p, g in zip(b, grads):
        p.grad = g
    ob.step()
    for p, q in zip(a, b):
        assert torch.equal(p, q)
    with pytest.raises(P.OptimError):
        P.opt_step(oa, grads[:1])
    with pytest.raises(P.OptimError):
        P.opt_step(oa, [grads[1], grads[0]])
