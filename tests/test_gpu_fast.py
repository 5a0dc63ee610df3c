"""GPU parity of the fast (tensor-core) path against the oracle, within the
fp32 tolerance the north star states:

  * one step: |theta_gpu - theta_ref| <= 1e-5 * (1 + |theta_ref|) elementwise
    (the reference's own cross-path bound, test_engine.py:262-275), states
    bitwise (the accumulator advance is exact in both modes);
  * 100 steps: relative L2 of the params <= 1e-5 (the reference's own
    naive-vs-fused drift is 2e-7), states bitwise.
"""

import numpy as np
import pytest

from conftest import F32, advanced_state, load_golden

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(scope="module")
def P():
    import torch

    assert torch.cuda.is_available()
    import paper_2506_10315_b200 as P

    assert P.fast_available(), "library built without the fast path"
    return P


def _close(got, want, tol=TOL):
    got = np.asarray(got, np.float64).reshape(-1)
    want = np.asarray(want, np.float64).reshape(-1)
    err = np.abs(got - want) / (1.0 + np.abs(want))
    return float(err.max()) if err.size else 0.0


ENGINE_SHAPES = [(1, 1), (1, 130), (130, 1), (5, 64), (7, 63), (3, 65), (33, 70), (64, 64),
                 (17, 129)]


@pytest.mark.parametrize("spec_name", ["small_fc_lopt", "velo_mlp"])
@pytest.mark.parametrize("shape", ENGINE_SHAPES)
def test_step_fused_fast_vs_reference_golden(P, oracle, spec_name, shape):
    import torch

    G = load_golden("engine_cases.npz")
    m, n = shape
    key = f"{spec_name}/{m}x{n}"
    s = oracle.OState.zeros(m, n)
    for i in range(3):
        s.M[i] = G[f"{key}/M{i}"]
        s.r[i] = G[f"{key}/r{i}"]
        s.c[i] = G[f"{key}/c{i}"]
    s.V = G[f"{key}/V"]
    s.t = int(G[f"{key}/t"][0])
    spec = P.spec_by_name(spec_name)
    W = torch.from_numpy(G[key + "/W"]).cuda()
    g = torch.from_numpy(G[key + "/g"]).cuda()
    w = P.random_weights(spec.d_feat, seed=int(G[key + "/wseed"][0]))
    st = P.DeviceOptState.from_arrays(s.M, s.V, s.r, s.c, s.t)
    sumsq, _ = P.fused_stats(W, g, st, spec, mode="fast")
    np.testing.assert_allclose(sumsq.cpu().numpy(), G[key + "/sumsq_w1"], rtol=2e-6)
    for lr in (1.0, 0.3):
        st = P.DeviceOptState.from_arrays(s.M, s.V, s.r, s.c, s.t)
        out, rep = P.step_fused(W, g, st, w, spec, lr=lr, mode="fast")
        err = _close(out.cpu().numpy(), G[key + f"/out_lr{lr}"])
        assert err <= TOL, err


@pytest.mark.parametrize("spec_name", ["small_fc_lopt", "velo_mlp"])
@pytest.mark.parametrize("shape", [(1, 1), (130, 1), (7, 63), (33, 70), (17, 129)])
def test_step_naive_vs_reference_naive_golden(P, oracle, spec_name, shape):
    """engine.step_naive (the non-bitwise class, here the tensor-core path)
    against the reference's own step_naive outputs (BLAS MLP), within the
    reference's cross-path bound 1e-5 (1 + |W|) (test_engine.py:262-275)."""
    import torch

    G = load_golden("engine_cases.npz")
    m, n = shape
    key = f"{spec_name}/{m}x{n}"
    s = oracle.OState.zeros(m, n)
    for i in range(3):
        s.M[i] = G[f"{key}/M{i}"]
        s.r[i] = G[f"{key}/r{i}"]
        s.c[i] = G[f"{key}/c{i}"]
    s.V = G[f"{key}/V"]
    s.t = int(G[f"{key}/t"][0])
    spec = P.spec_by_name(spec_name)
    W = torch.from_numpy(G[key + "/W"]).cuda()
    g = torch.from_numpy(G[key + "/g"]).cuda()
    w = P.random_weights(spec.d_feat, seed=int(G[key + "/wseed"][0]))
    for lr in (1.0, 0.3):
        st = P.DeviceOptState.from_arrays(s.M, s.V, s.r, s.c, s.t)
        out, _ = P.step_naive(W, g, st, w, spec, lr=lr)
        ref = G[key + f"/naive_lr{lr}"].astype(np.float64)
        err = (np.abs(out.cpu().numpy().astype(np.float64) - ref) / (1 + np.abs(ref))).max()
        assert err <= 1e-5, err


SHAPE_SETS = {
    "mlp": [(128, 784), (128,), (10, 128), (10,)],
    "vit_block": [(2304, 768), (2304,), (768, 768), (768,), (3072, 768), (768, 3072), (1, 197, 768),
                  (768, 3, 16, 16), (1, 1, 768)],
    "odd": [(33, 70), (1, 130), (130, 1), (7, 63), (1000, 3), (5,), ()],
}


@pytest.mark.parametrize("feature_set", ["small_fc_lopt", "velo_mlp"])
@pytest.mark.parametrize("which", ["mlp", "vit_block", "odd"])
def test_fast_optimizer_steps_vs_oracle(P, oracle, feature_set, which):
    import torch

    shapes = SHAPE_SETS[which]
    rng = np.random.default_rng(5)
    init = [np.asarray(rng.standard_normal(s) * 0.02, dtype=F32) for s in shapes]
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, feature_set=feature_set, mode="fast", weight_decay=0.01)
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [oracle.OState.zeros(*p.shape) for p in o_params]
    kind = oracle.KIND_BY_NAME[feature_set]
    w = oracle.random_weights(39 if kind == oracle.SMALL_FC_LOPT else 29, seed=0)
    worst = 0.0
    for step in range(3):
        grads = [(rng.standard_normal(p.shape) * 1e-3).astype(F32) for p in o_params]
        # make the next step start from identical params (tolerance, not drift)
        for p, q in zip(params, o_params):
            p.data.copy_(torch.from_numpy(q.reshape(p.shape)).cuda())
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step()
        oracle.opt_step(o_params, o_states, grads, w, kind, 1.0, weight_decay=0.01, threads=8)
        for p, q in zip(params, o_params):
            worst = max(worst, _close(p.detach().cpu().numpy(), q))
    print(f"max elementwise err/(1+|theta|) {which} {feature_set}: {worst:.3e}")
    assert worst <= TOL, worst
    for p, s in zip(params, o_states):
        quad = opt.state[p]["quad"].cpu().numpy()
        assert quad[:, 3].tobytes() == s.V.reshape(-1).tobytes()
        assert quad[:, 2].tobytes() == s.M[2].reshape(-1).tobytes()
        assert opt.state[p]["row_factors"].cpu().numpy()[1].tobytes() == s.r[1].tobytes()
        assert opt.state[p]["col_factors"].cpu().numpy()[2].tobytes() == s.c[2].tobytes()


@pytest.mark.parametrize("feature_set", ["small_fc_lopt", "velo_mlp"])
def test_fast_hundred_steps_relative_l2(P, oracle, feature_set):
    """Free-running trajectories (no re-sync) on the MNIST-shaped MLP with a
    cosine schedule and decay: relative L2 of the params after 100 steps."""
    import torch

    shapes = [(128, 784), (128,), (10, 128), (10,)]
    rng = np.random.default_rng(11)
    init = [(rng.standard_normal(s) * 0.05).astype(F32) for s in shapes]
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, feature_set=feature_set, weight_decay=0.01, mode="fast",
                             schedule=P.ScheduleConfig("cosine", 0.5, 0.01, 5, 100))
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [oracle.OState.zeros(*p.shape) for p in o_params]
    kind = oracle.KIND_BY_NAME[feature_set]
    w = oracle.random_weights(39 if kind == oracle.SMALL_FC_LOPT else 29, seed=0)
    for step in range(100):
        grads = [(rng.standard_normal(p.shape) * 1e-2).astype(F32) for p in o_params]
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step()
        lr = oracle.schedule_lr("cosine", 0.5, 0.01, 5, 100, step)
        oracle.opt_step(o_params, o_states, grads, w, kind, lr, weight_decay=0.01)
    for p, q in zip(params, o_params):
        got = p.detach().cpu().numpy().reshape(-1).astype(np.float64)
        want = q.reshape(-1).astype(np.float64)
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        print(f"100-step relL2 {feature_set} {p.shape}: {rel:.3e}")
        assert rel <= 2e-6, rel
    for p, s in zip(params, o_states):
        quad = opt.state[p]["quad"].cpu().numpy()
        assert quad[:, 0].tobytes() == s.M[0].reshape(-1).tobytes()


def test_fast_nonfinite_gradient_raises(P):
    import torch

    a = torch.nn.Parameter(torch.ones(256, 128, device="cuda"))
    opt = P.LearnedOptimizer([a], mode="fast")
    g = torch.ones(256, 128, device="cuda")
    g[3, 7] = float("inf")
    a.grad = g
    with pytest.raises(P.OptimError):
        opt.step()
    assert torch.equal(a.detach(), torch.ones(256, 128, device="cuda"))


def test_fast_zero_network_is_noop(P):
    import torch

    x = torch.randn(300, 256, device="cuda")
    p = torch.nn.Parameter(x.clone())
    opt = P.LearnedOptimizer([p], weights=P.zero_weights(39), mode="fast")
    p.grad = torch.randn(300, 256, device="cuda")
    opt.step()
    assert torch.equal(p.detach(), x)


@pytest.mark.parametrize("mode", ["strict", "fast"])
@pytest.mark.parametrize("flat_host", [False, True])
def test_step_host_matches_device_step(P, mode, flat_host):
    """step_host (chunked H2D / step / D2H pipeline) gives the same parameters
    and state as step() on device-resident gradients -- bitwise, since both
    run the same kernels on the same tensors.  flat_host: the host tensors are
    consecutive views of one pinned buffer, so each tensor group moves as one
    copy; otherwise per-tensor copies."""
    import torch

    shapes = [(128, 784), (128,), (10, 128), (10,), (256, 256), (33, 70)]
    rng = np.random.default_rng(11)
    init = [np.asarray(rng.standard_normal(s) * 0.02, dtype=F32) for s in shapes]
    grads = [[np.asarray(rng.standard_normal(s) * 1e-3, dtype=F32) for s in shapes]
             for _ in range(3)]
    a = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    b = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    oa = P.LearnedOptimizer(a, mode=mode, weight_decay=0.01)
    ob = P.LearnedOptimizer(b, mode=mode, weight_decay=0.01)
    sizes = [int(np.prod(s)) for s in shapes]
    offs = np.cumsum([0] + sizes)

    def host_views(buf):
        return [buf[offs[k]:offs[k + 1]].view(s) for k, s in enumerate(shapes)]

    if flat_host:
        host_p = host_views(torch.empty(offs[-1], dtype=torch.float32).pin_memory())
    else:
        host_p = [torch.empty(s, dtype=torch.float32).pin_memory() for s in shapes]
    for gs in grads:
        for p, g in zip(a, gs):
            p.grad = torch.from_numpy(g).cuda()
        oa.step()
        if flat_host:
            hg = host_views(torch.from_numpy(np.concatenate([g.reshape(-1) for g in gs])).pin_memory())
        else:
            hg = [torch.from_numpy(g).pin_memory() for g in gs]
        ob.step_host(hg, host_p, chunks=3)
    from paper_2506_10315_b200.optim import _flat_host_view

    assert (_flat_host_view(host_p, b) is not None) == flat_host
    torch.cuda.synchronize()
    for p, q, h in zip(a, b, host_p):
        assert p.detach().cpu().numpy().tobytes() == q.detach().cpu().numpy().tobytes()
        assert h.numpy().tobytes() == q.detach().cpu().numpy().tobytes()
    for p, q in zip(a, b):
        assert oa.state[p]["quad"].cpu().numpy().tobytes() == ob.state[q]["quad"].cpu().numpy().tobytes()


def test_fused_peer_copies_single_gpu(P):
    """The fused all-gather path with stand-in peers: two more arenas on the
    same device play the other ranks' parameter copies; after a fast step they
    must hold exactly the updated parameters (same kernel stores, other
    addresses), and the local result must equal a step without peers."""
    import torch

    shapes = [(128, 784), (128,), (10, 128), (10,), (33, 70)]
    total = sum(int(np.prod(s)) for s in shapes)
    rng = np.random.default_rng(4)
    init = [np.asarray(rng.standard_normal(s) * 0.02, dtype=F32) for s in shapes]
    grads = [np.asarray(rng.standard_normal(s) * 1e-3, dtype=F32) for s in shapes]

    def build(arena):
        ps, off = [], 0
        for x, s in zip(init, shapes):
            n = x.size
            arena[off:off + n].copy_(torch.from_numpy(x.reshape(-1)))
            ps.append(torch.nn.Parameter(arena[off:off + n].view(s)))
            off += n
        return ps

    arena = torch.zeros(total, device="cuda")
    peers = [torch.full((total,), 7.0, device="cuda") for _ in range(2)]
    ps = build(arena)
    opt = P.LearnedOptimizer(ps, mode="fast", weight_decay=0.01)
    opt.set_peer_copies([q.data_ptr() - arena.data_ptr() for q in peers])
    for p, g in zip(ps, grads):
        p.grad = torch.from_numpy(g).cuda()
    opt.step()
    ref_arena = torch.zeros(total, device="cuda")
    rs = build(ref_arena)
    ropt = P.LearnedOptimizer(rs, mode="fast", weight_decay=0.01)
    for p, g in zip(rs, grads):
        p.grad = torch.from_numpy(g).cuda()
    ropt.step()
    torch.cuda.synchronize()
    assert torch.equal(arena, ref_arena)
    for q in peers:
        assert torch.equal(q, arena)


@pytest.mark.parametrize("b2_shift", [-3.0, 3.0])
def test_fast_layer3_split_accuracy_with_skewed_hidden_layer(P, oracle, b2_shift):
    """The fast epilogue forms relu(h2).w3 as 1/2 w3.h2 (on the tensor cores,
    layer-2 extra rows) + 1/2 w3.|h2| (FFMA2).  A layer-2 bias pushed far
    negative makes most h2 < 0, so the two halves nearly cancel; pushed
    positive, relu is the identity.  Both stay inside the reference's
    cross-path bound 1e-5 (1 + |theta|)."""
    import torch

    shapes = [(128, 784), (128,), (10, 128), (10,), (33, 70)]
    rng = np.random.default_rng(21)
    init = [np.asarray(rng.standard_normal(s) * 0.02, dtype=F32) for s in shapes]
    ow = oracle.random_weights(39, seed=3)
    layers = [(w.copy(), b.copy()) for w, b in ow.layers]
    w2, b2 = layers[1]
    layers[1] = (w2, (b2 + np.float32(b2_shift)).astype(F32))
    w3, b3 = layers[2]
    layers[2] = ((w3 * np.float32(4.0)).astype(F32), b3)
    ow.layers = layers
    pw = P.LoptWeights(layers=[(w.copy(), b.copy()) for w, b in layers])
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, mode="fast", weights=pw)
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [oracle.OState.zeros(*p.shape) for p in o_params]
    worst = 0.0
    for step in range(2):
        grads = [(rng.standard_normal(p.shape) * 1e-3).astype(F32) for p in o_params]
        for p, q in zip(params, o_params):
            p.data.copy_(torch.from_numpy(q.reshape(p.shape)).cuda())
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step()
        oracle.opt_step(o_params, o_states, grads, ow, oracle.SMALL_FC_LOPT, 1.0, threads=8)
        for p, q in zip(params, o_params):
            worst = max(worst, _close(p.detach().cpu().numpy(), q))
    print(f"b2 shift {b2_shift}: max err/(1+|theta|) {worst:.3e}")
    assert worst <= TOL, worst


def test_step_host_accepts_numpy_arrays(P):
    """The reference's calling convention: gradients in, parameters out as
    NumPy arrays (wrapped without a copy; synchronous transfers)."""
    import torch

    shapes = [(64, 96), (64,), (33, 70)]
    rng = np.random.default_rng(17)
    init = [np.asarray(rng.standard_normal(s) * 0.02, dtype=F32) for s in shapes]
    grads = [np.asarray(rng.standard_normal(s) * 1e-3, dtype=F32) for s in shapes]
    a = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    b = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    oa = P.LearnedOptimizer(a, mode="fast")
    ob = P.LearnedOptimizer(b, mode="fast")
    for p, g in zip(a, grads):
        p.grad = torch.from_numpy(g).cuda()
    oa.step()
    out = [np.empty(s, F32) for s in shapes]
    ob.step_host(grads, out, chunks=2)
    torch.cuda.synchronize()
    for p, h in zip(a, out):
        assert p.detach().cpu().numpy().tobytes() == h.tobytes()


@pytest.mark.parametrize("n_peers", [1, 7])
def test_fused_peer_bulk_copies_model_shapes(P, n_peers):
    """Bulk (TMA) peer copies of whole tiles: ViT-like aligned shapes with
    many tiles per CTA (both staging buffers cycle), up to LOPT_MAX_PEERS
    stand-in peers; every peer arena must equal the stepped local arena."""
    import torch

    shapes = [(768, 768), (2304,), (768, 3072), (197, 768), (1000,), (5, 7)]
    total = sum(int(np.prod(s)) for s in shapes)
    rng = np.random.default_rng(11)
    arena = torch.zeros(total, device="cuda")
    ps, off = [], 0
    for s in shapes:
        n = int(np.prod(s))
        arena[off:off + n].copy_(torch.from_numpy(np.asarray(rng.standard_normal(n) * 0.02, F32)))
        ps.append(torch.nn.Parameter(arena[off:off + n].view(s)))
        off += n
    ref = arena.clone()
    peers = [torch.full((total,), -3.0, device="cuda") for _ in range(n_peers)]
    opt = P.LearnedOptimizer(ps, mode="fast")
    opt.set_peer_copies([q.data_ptr() - arena.data_ptr() for q in peers])
    rps, off = [], 0
    for s in shapes:
        n = int(np.prod(s))
        rps.append(torch.nn.Parameter(ref[off:off + n].view(s)))
        off += n
    ropt = P.LearnedOptimizer(rps, mode="fast")
    for step in range(2):
        for p, q in zip(ps, rps):
            g = torch.from_numpy(np.asarray(rng.standard_normal(p.shape) * 1e-3, F32)).cuda()
            p.grad, q.grad = g, g.clone()
        opt.step()
        ropt.step()
    torch.cuda.synchronize()
    assert torch.equal(arena, ref)
    for q in peers:
        assert torch.equal(q, arena)
