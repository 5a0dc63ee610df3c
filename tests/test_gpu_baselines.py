"""The reference's baseline optimizers on the device (paper_2506_10315_b200.baselines)
against the reference's own outputs (tests/golden/baseline_cases.npz, made by
gen_baselines.py) and the oracle at model sizes: Adam bitwise; Adafactor's
factors within 1 f32 ulp (its f64 means use a fixed device order instead of
numpy's), the parameters within that ulp's effect on the update."""

import numpy as np
import pytest
import torch

from conftest import load_golden

F32 = np.float32
B = load_golden("baseline_cases.npz")


def _ulps(a, b):
    ia = a.view(np.int32).astype(np.int64)
    ib = b.view(np.int32).astype(np.int64)
    return np.abs(ia - ib)


def test_baselines_refuse_host_tensors_and_bad_t():
    from paper_2506_10315_b200.baselines import adafactor_step, adam_step

    x = torch.zeros(2, 2)
    with pytest.raises(ValueError):
        adam_step(x, x, x, x, t=0)
    with pytest.raises(TypeError):
        adam_step(x, x, x, x, t=1)
    with pytest.raises(TypeError):
        adafactor_step(x, x, torch.zeros(2), torch.zeros(2))


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(4))
def test_adam_bitwise_vs_reference(k):
    from paper_2506_10315_b200.baselines import adam_step

    th = torch.from_numpy(B[f"adam{k}/theta0"].copy()).cuda()
    m, v = torch.zeros_like(th), torch.zeros_like(th)
    for t in range(1, 5):
        g = torch.from_numpy(B[f"adam{k}/g{t}"].copy()).cuda()
        adam_step(th, g, m, v, lr=1e-3 if t != 3 else 0.05, t=t)
        for nm, x in (("theta", th), ("m", m), ("v", v)):
            got = x.cpu().numpy()
            assert np.array_equal(got.view(np.uint32), B[f"adam{k}/{nm}{t}"].view(np.uint32)), (nm, t)


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(5))
def test_adafactor_vs_reference(k):
    from paper_2506_10315_b200.baselines import adafactor_step

    th = torch.from_numpy(B[f"afac{k}/theta0"].copy()).cuda()
    r = torch.zeros(th.shape[0], device="cuda")
    c = torch.zeros(th.shape[1], device="cuda")
    for t in range(1, 4):
        g = torch.from_numpy(B[f"afac{k}/g{t}"].copy()).cuda()
        lr = 1e-2 if t == 2 else 1e-3
        prev = th.clone()
        adafactor_step(th, g, r, c, lr=lr)
        assert _ulps(r.cpu().numpy(), B[f"afac{k}/r{t}"]).max() <= 1
        assert _ulps(c.cpu().numpy(), B[f"afac{k}/c{t}"]).max() <= 1
        want = B[f"afac{k}/theta{t}"]
        upd = np.abs(want - prev.cpu().numpy())
        assert np.all(np.abs(th.cpu().numpy() - want) <= 4e-7 * upd + 1e-30 + np.spacing(np.abs(want)))
        # continue from the reference's values so errors do not compound
        th.copy_(torch.from_numpy(want))
        r.copy_(torch.from_numpy(B[f"afac{k}/r{t}"]))
        c.copy_(torch.from_numpy(B[f"afac{k}/c{t}"]))


@pytest.mark.gpu
@pytest.mark.parametrize("shape", [(3072, 768), (768, 1), (2304, 768)])
def test_baselines_model_size_vs_oracle(oracle, shape):
    from paper_2506_10315_b200.baselines import adafactor_step, adam_step

    rng = np.random.default_rng(7)
    th0 = (rng.standard_normal(shape) * 0.02).astype(F32)
    g = (rng.standard_normal(shape) * 1e-3).astype(F32)
    m0 = (rng.standard_normal(shape) * 1e-4).astype(F32)
    v0 = np.abs(rng.standard_normal(shape) * 1e-6).astype(F32)
    want = oracle.adam_step(th0, g, m0, v0, lr=1e-3, t=3)
    th, gd = torch.from_numpy(th0.copy()).cuda(), torch.from_numpy(g).cuda()
    m, v = torch.from_numpy(m0.copy()).cuda(), torch.from_numpy(v0.copy()).cuda()
    adam_step(th, gd, m, v, lr=1e-3, t=3)
    for x, w in zip((th, m, v), want):
        assert np.array_equal(x.cpu().numpy().view(np.uint32), w.view(np.uint32))
    r0 = np.abs(rng.standard_normal(shape[0]) * 1e-6).astype(F32)
    c0 = np.abs(rng.standard_normal(shape[1]) * 1e-6).astype(F32)
    wt, wr, wc = oracle.adafactor_step(th0, g, r0, c0, lr=1e-3)
    th = torch.from_numpy(th0.copy()).cuda()
    r, c = torch.from_numpy(r0.copy()).cuda(), torch.from_numpy(c0.copy()).cuda()
    adafactor_step(th, gd, r, c, lr=1e-3)
    assert _ulps(r.cpu().numpy(), wr).max() <= 1
    assert _ulps(c.cpu().numpy(), wc).max() <= 1
    upd = np.abs(wt - th0)
    assert np.all(np.abs(th.cpu().numpy() - wt) <= 4e-7 * upd + np.spacing(np.abs(wt)))
