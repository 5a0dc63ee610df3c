"""Parity at the benchmark's full sizes through properties that do not need
the (slow) CPU reference: strict mode is bitwise equal to the reference on
every fixture (test_gpu_strict.py), so fast-vs-strict on the full ViT-B/16
parameter census and on GPT-2 medium's largest tensor (wte, 51.5 M elements)
is fast-vs-reference at full size.  Accumulators and factors must agree bit
for bit, parameters within the fp32 tolerance, and the per-tensor max |delta|
reports must agree."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
TOL = 1e-5


def _census(name):
    from paper_2506_10315_b200.workloads import WORKLOADS
    return [s for _, s in WORKLOADS[name]()]


def _run(shapes, fs, steps, seed=0):
    import torch

    import paper_2506_10315_b200 as P

    g = torch.Generator(device="cpu").manual_seed(seed)
    init = [torch.empty(s).normal_(0, 0.02, generator=g) for s in shapes]
    grads = [[torch.empty(s).normal_(0, 1e-3, generator=g) for s in shapes] for _ in range(steps)]
    out = {}
    for mode in ("strict", "fast"):
        ps = [torch.nn.Parameter(x.clone().cuda()) for x in init]
        opt = P.LearnedOptimizer(ps, feature_set=fs, mode=mode, weight_decay=0.01)
        for k in range(steps):
            for p, gr in zip(ps, grads[k]):
                p.grad = gr.cuda()
            opt.step()
        torch.cuda.synchronize()
        out[mode] = (ps, opt)
    return out


@pytest.mark.parametrize("fs", ["small_fc_lopt", "velo_mlp"])
def test_vit_b16_fast_equals_strict(fs):
    import torch

    out = _run(_census("vit_b16"), fs, steps=2)
    (ps_s, opt_s), (ps_f, opt_f) = out["strict"], out["fast"]
    worst = 0.0
    for a, b in zip(ps_s, ps_f):
        sa, sb = opt_s.state[a], opt_f.state[b]
        assert torch.equal(sa["quad"], sb["quad"])
        assert torch.equal(sa["row_factors"], sb["row_factors"])
        assert torch.equal(sa["col_factors"], sb["col_factors"])
        err = ((b.detach() - a.detach()).abs() / (1 + a.detach().abs())).max().item()
        worst = max(worst, err)
    assert worst <= TOL, worst
    ma, mb = np.array(opt_s.max_abs_updates()), np.array(opt_f.max_abs_updates())
    assert np.allclose(ma, mb, rtol=1e-4, atol=1e-9)


def test_gpt2_wte_fast_equals_strict():
    import torch

    shapes = [(50257, 1024), (1024,)]
    out = _run(shapes, "velo_mlp", steps=1, seed=1)
    (ps_s, opt_s), (ps_f, opt_f) = out["strict"], out["fast"]
    for a, b in zip(ps_s, ps_f):
        assert torch.equal(opt_s.state[a]["quad"], opt_f.state[b]["quad"])
        err = ((b.detach() - a.detach()).abs() / (1 + a.detach().abs())).max().item()
        assert err <= TOL, err


def _vit_block_subset():
    """One ViT-B/16 encoder block + conv_proj + pos_embedding (7.8 M params)."""
    names = ("conv_proj", "encoder.pos_embedding", "encoder_layer_0.")
    from paper_2506_10315_b200.workloads import vit_b16
    return [s for n, s in vit_b16() if any(k in n for k in names)]


@pytest.mark.parametrize("feature_set", ["small_fc_lopt", "velo_mlp"])
def test_vit_subset_hundred_steps_relative_l2_vs_oracle(oracle, feature_set):
    """BASELINE.md section 4(5) / north_star: 100 free-running fast-mode steps
    on a >= 5 M-param ViT-B/16 subset (encoder block 0, conv_proj,
    pos_embedding) against the CPU oracle (bitwise the reference), cosine
    schedule + decay; relative L2 of the parameters <= 2e-6 and the
    accumulators bitwise."""
    import torch

    import paper_2506_10315_b200 as P

    shapes = _vit_block_subset()
    assert sum(int(np.prod(s)) for s in shapes) >= 5_000_000
    rng = np.random.default_rng(21)
    init = [(rng.standard_normal(s, dtype=np.float32) * 0.02) for s in shapes]
    params = [torch.nn.Parameter(torch.from_numpy(x.copy()).cuda()) for x in init]
    opt = P.LearnedOptimizer(params, feature_set=feature_set, weight_decay=0.01, mode="fast",
                             schedule=P.ScheduleConfig("cosine", 0.5, 0.01, 5, 100))
    o_params = [x.reshape(P.view_2d(x.shape)).copy() for x in init]
    o_states = [oracle.OState.zeros(*p.shape) for p in o_params]
    kind = oracle.KIND_BY_NAME[feature_set]
    w = oracle.random_weights(39 if kind == oracle.SMALL_FC_LOPT else 29, seed=0)
    for step in range(100):
        grads = [rng.standard_normal(p.shape, dtype=np.float32) * np.float32(1e-3)
                 for p in o_params]
        for p, g in zip(params, grads):
            p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
        opt.step()
        lr = oracle.schedule_lr("cosine", 0.5, 0.01, 5, 100, step)
        oracle.opt_step(o_params, o_states, grads, w, kind, lr, weight_decay=0.01)
    worst = 0.0
    for p, q in zip(params, o_params):
        got = p.detach().cpu().numpy().reshape(-1).astype(np.float64)
        want = q.reshape(-1).astype(np.float64)
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        worst = max(worst, rel)
    print(f"100-step relL2 {feature_set} ViT subset: worst {worst:.3e}")
    assert worst <= 2e-6, worst
    for p, s in zip(params, o_states):
        quad = opt.state[p]["quad"].cpu().numpy()
        assert quad[:, 0].tobytes() == s.M[0].reshape(-1).tobytes()
        assert quad[:, 3].tobytes() == s.V.reshape(-1).tobytes()
        assert opt.state[p]["row_factors"].cpu().numpy().tobytes() == np.stack(s.r).tobytes()
        assert opt.state[p]["col_factors"].cpu().numpy().tobytes() == np.stack(s.c).tobytes()


def test_gpt2_medium_velo_cosine_wd_full_census_fast_equals_strict():
    """BASELINE.json config 5 on the whole GPT-2 medium census (292 tensors,
    354.8 M params): VeLO_CUDA (per-tensor LSTM hypernetwork) with a cosine
    schedule and weight decay 0.01, 3 steps in fast and in strict mode (strict
    is bitwise the reference's per-element path, test_gpu_strict.py):
    accumulators and factors bitwise, parameters within the fp32 tolerance."""
    import torch

    import paper_2506_10315_b200 as P

    shapes = _census("gpt2_medium")
    sched = P.ScheduleConfig("cosine", 1.0, 0.1, 2, 10_000)
    out = {}
    for mode in ("strict", "fast"):
        g = torch.Generator(device="cuda").manual_seed(5)
        ps = [torch.nn.Parameter(torch.empty(s, device="cuda").normal_(0, 0.02, generator=g))
              for s in shapes]
        opt = P.VeLO_CUDA(ps, mode=mode, weight_decay=0.01, schedule=sched,
                          hypernet=P.VeLOHyperNet(seed=2))
        for k in range(3):
            for p in ps:
                p.grad = torch.empty_like(p).normal_(0, 1e-3, generator=g)
            opt.step(loss=3.0 - 0.2 * k)
        torch.cuda.synchronize()
        out[mode] = (ps, opt)
        for p in ps:
            p.grad = None
    (ps_s, opt_s), (ps_f, opt_f) = out["strict"], out["fast"]
    worst = 0.0
    for a, b in zip(ps_s, ps_f):
        sa, sb = opt_s.state[a], opt_f.state[b]
        assert torch.equal(sa["quad"], sb["quad"])
        assert torch.equal(sa["row_factors"], sb["row_factors"])
        assert torch.equal(sa["col_factors"], sb["col_factors"])
        err = ((b.detach() - a.detach()).abs() / (1 + a.detach().abs())).max().item()
        worst = max(worst, err)
    print(f"gpt2-medium VeLO 3-step fast vs strict: worst {worst:.3e}")
    assert worst <= TOL, worst
