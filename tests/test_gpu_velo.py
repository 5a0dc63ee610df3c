"""VeLO on the GPU: the per-tensor LSTM hypernetwork kernel against its numpy
restatement (oracle/velo_lstm.py, self-pinned: the reference has no VeLO
LSTM), and the full VeLO step against the oracle driven with the mixed
per-tensor MLPs (the per-element half is the reference's VELO_MLP path)."""

import numpy as np
import pytest

from conftest import F32

pytestmark = pytest.mark.gpu

SHAPES = [(256, 192), (256,), (96, 256), (96,), (33, 70), (7,)]


def _setup(P, mode, K=4, seed=3):
    import torch

    rng = np.random.default_rng(seed)
    init = [np.asarray(rng.standard_normal(s) * 0.05, F32) for s in SHAPES]
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    hn = P.VeLOHyperNet(hidden=16, bank_size=K, seed=seed)
    opt = P.VeLO_CUDA(params, weight_decay=0.01, hypernet=hn, mode=mode)
    return rng, init, params, hn, opt


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_velo_step_matches_oracle_with_mixed_mlps(oracle, mode):
    import torch

    import paper_2506_10315_b200 as P
    from oracle import velo_lstm as V

    rng, init, params, hn, opt = _setup(P, mode)
    opt._mix_out = torch.zeros(len(params), hn.K, device="cuda")
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [oracle.OState.zeros(*p.shape) for p in o_params]
    lstm = np.zeros((len(params), 2 * hn.H), F32)
    bank = hn.packed_bank()
    ema = None
    for step in range(4):
        grads = [np.asarray(rng.standard_normal(p.shape) * 1e-2, F32) for p in o_params]
        loss = 2.0 / (1 + step)
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step(loss=loss)
        # oracle: the merged sums are the GPU's (phase 1 is covered by the
        # engine tests); the hypernetwork is the numpy restatement
        sumsq = opt.plans()[0].stat_sums().cpu().numpy()
        counts = np.array([p.shape[0] * p.shape[1] for p in o_params])
        lf, ema = V.loss_features(loss, ema)
        mixed, alphas, lstm = V.velo_mix(hn.hyper, lstm, bank, sumsq, counts, step + 1, lf,
                                         H=hn.H, K=hn.K)
        np.testing.assert_allclose(opt._mix_out.cpu().numpy(), alphas, rtol=1e-5, atol=1e-6)
        gpu_lstm = opt._lstm[0][0].cpu().numpy()
        np.testing.assert_allclose(gpu_lstm, lstm, rtol=1e-5, atol=1e-6)
        lstm = gpu_lstm.copy()   # continue from the device state (tolerance, not drift)
        ws = [P.weights.unpack(m, 29) for m in mixed]
        ow = [oracle.Weights(layers=w.layers) for w in ws]
        oracle.opt_step(o_params, o_states, grads, ow[0], oracle.VELO_MLP, 1.0,
                        weight_decay=0.01, per_tensor_weights=ow)
        worst = 0.0
        for p, q in zip(params, o_params):
            got = p.detach().cpu().numpy().reshape(-1).astype(np.float64)
            want = q.reshape(-1)
            worst = max(worst, float(np.max(np.abs(got - want) / (1 + np.abs(want)))))
            p.data.copy_(torch.from_numpy(q.reshape(p.shape)).cuda())
        assert worst <= 1e-5, (step, worst)


def test_velo_bank_of_one_is_the_velo_mlp_step(oracle):
    """A one-MLP bank mixes to that MLP exactly: VeLO_CUDA == the reference's
    VELO_MLP step with that MLP, bit for bit in strict mode."""
    import torch

    import paper_2506_10315_b200 as P

    rng = np.random.default_rng(0)
    init = [np.asarray(rng.standard_normal(s) * 0.05, F32) for s in SHAPES]
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    hn = P.VeLOHyperNet(hidden=8, bank_size=1, seed=1)
    opt = P.VeLO_CUDA(params, hypernet=hn, mode="strict")
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [oracle.OState.zeros(*p.shape) for p in o_params]
    ow = oracle.Weights(layers=hn.bank[0].layers)
    for step in range(3):
        grads = [np.asarray(rng.standard_normal(p.shape) * 1e-2, F32) for p in o_params]
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step(loss=1.0)
        oracle.opt_step(o_params, o_states, grads, ow, oracle.VELO_MLP, 1.0)
    for p, q in zip(params, o_params):
        assert p.detach().cpu().numpy().reshape(-1).tobytes() == q.reshape(-1).tobytes()


def test_velo_requires_loss():
    import torch

    import paper_2506_10315_b200 as P

    p = torch.nn.Parameter(torch.ones(4, 4, device="cuda"))
    opt = P.VeLO_CUDA([p])
    p.grad = torch.ones(4, 4, device="cuda")
    with pytest.raises(P.OptimError):
        opt.step()


def test_velo_step_host_matches_device_step():
    """VeLO through the host-buffer step (tensor groups, each running the
    hypernetwork between its phases) equals VeLO_CUDA.step on device-resident
    gradients bit for bit: the per-tensor LSTM and the per-element kernels do
    not depend on how tensors are grouped."""
    import torch

    import paper_2506_10315_b200 as P

    shapes = [(128, 784), (128,), (10, 128), (10,), (33, 70)]
    rng = np.random.default_rng(13)
    init = [np.asarray(rng.standard_normal(s) * 0.02, dtype=np.float32) for s in shapes]
    grads = [[np.asarray(rng.standard_normal(s) * 1e-3, dtype=np.float32) for s in shapes]
             for _ in range(3)]
    a = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    b = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    oa = P.VeLO_CUDA(a, mode="fast", weight_decay=0.01)
    ob = P.VeLO_CUDA(b, mode="fast", weight_decay=0.01)
    host_p = [torch.empty(s, dtype=torch.float32).pin_memory() for s in shapes]
    for k, gs in enumerate(grads):
        for p, g in zip(a, gs):
            p.grad = torch.from_numpy(g).cuda()
        oa.step(loss=2.0 - 0.1 * k)
        ob.step_host([torch.from_numpy(g).pin_memory() for g in gs], host_p, chunks=2,
                     loss=2.0 - 0.1 * k)
    torch.cuda.synchronize()
    for p, q, h in zip(a, b, host_p):
        assert p.detach().cpu().numpy().tobytes() == q.detach().cpu().numpy().tobytes()
        assert h.numpy().tobytes() == q.detach().cpu().numpy().tobytes()


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_velo_state_dict_resume_is_bitwise(mode):
    """VeLO checkpoint/resume: the per-tensor LSTM state and the loss EMA
    travel in state_dict, so a fresh optimizer loaded mid-run continues the
    trajectory bit for bit."""
    import copy

    import torch

    import paper_2506_10315_b200 as P

    shapes = [(64, 96), (64,), (10, 64), (10,)]
    rng = np.random.default_rng(3)
    init = [np.asarray(rng.standard_normal(s) * 0.02, dtype=np.float32) for s in shapes]
    grads = [[np.asarray(rng.standard_normal(s) * 1e-3, dtype=np.float32) for s in shapes]
             for _ in range(4)]
    losses = [2.0, 1.8, 1.7, 1.5]

    def run(opt, params, ks):
        for k in ks:
            for p, g in zip(params, grads[k]):
                p.grad = torch.from_numpy(g).cuda()
            opt.step(loss=losses[k])

    a = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    oa = P.VeLO_CUDA(a, mode=mode)
    run(oa, a, [0, 1])
    sd = copy.deepcopy(oa.state_dict())
    mid = [p.detach().clone() for p in a]
    run(oa, a, [2, 3])
    b = [torch.nn.Parameter(t.clone()) for t in mid]
    ob = P.VeLO_CUDA(b, mode=mode)
    ob.load_state_dict(sd)
    run(ob, b, [2, 3])
    torch.cuda.synchronize()
    for p, q in zip(a, b):
        assert p.detach().cpu().numpy().tobytes() == q.detach().cpu().numpy().tobytes()


@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_velo_nonfinite_gradient_changes_nothing_then_recovers(mode):
    """optim.py:160-165 for the whole VeLO step: a non-finite gradient raises
    OptimError and changes nothing -- parameters, accumulators, factors, the
    per-tensor LSTM state and the loss EMA -- and the next finite step equals
    the step of an optimizer that never saw the bad one (bitwise)."""
    import torch

    import paper_2506_10315_b200 as P

    rng, init, params, hn, opt = _setup(P, mode)
    ref = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt_ref = P.VeLO_CUDA(ref, weight_decay=0.01, hypernet=hn, mode=mode)
    g1 = [np.asarray(rng.standard_normal(p.shape) * 1e-2, F32) for p in init]
    g2 = [np.asarray(rng.standard_normal(p.shape) * 1e-2, F32) for p in init]
    for o, ps in ((opt, params), (opt_ref, ref)):
        for p, g in zip(ps, g1):
            p.grad = torch.from_numpy(g).cuda()
        o.step(loss=2.0)
    lstm0 = opt._lstm[0][0].clone()
    ema0 = opt._loss_ema
    theta0 = [p.detach().clone() for p in params]
    quad0 = [opt.state[p]["quad"].clone() for p in params]
    bad = [torch.from_numpy(g).cuda() for g in g2]
    bad[2].view(-1)[17] = float("inf")
    for p, g in zip(params, bad):
        p.grad = g
    with pytest.raises(P.OptimError):
        opt.step(loss=1.5)
    assert torch.equal(opt._lstm[0][0], lstm0)
    assert opt._loss_ema == ema0
    for p, t0, q0 in zip(params, theta0, quad0):
        assert torch.equal(p.detach(), t0)
        assert torch.equal(opt.state[p]["quad"], q0)
    for o, ps in ((opt, params), (opt_ref, ref)):
        for p, g in zip(ps, g2):
            p.grad = torch.from_numpy(g).cuda()
        o.step(loss=1.5)
    for a, b in zip(params, ref):
        assert torch.isfinite(a).all()
        assert torch.equal(a.detach(), b.detach())
    assert torch.equal(opt._lstm[0][0], opt_ref._lstm[0][0])
