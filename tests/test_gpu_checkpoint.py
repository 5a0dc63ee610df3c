"""Bitwise resume from a reference checkpoint (SURVEY.md section 8(f) rank 1,
acceptance 10): a checkpoint written by the reference after 3 steps is loaded
into the GPU optimizer, which continues for 2 steps on the reference's
gradients; parameters and accumulators must equal the reference's own
continuation bit for bit (strict mode) / within the fp32 tolerance (fast)."""

import os

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
GOLD = os.path.join(ROOT, "tests", "golden")


@pytest.mark.parametrize("run", ["small_const", "velo_cos_wd"])
@pytest.mark.parametrize("mode", ["strict", "fast"])
def test_resume_reference_checkpoint(run, mode):
    import torch

    from paper_2506_10315_b200 import container

    z = np.load(os.path.join(GOLD, "ckpt_cases.npz"))
    opt, params, names = container.checkpoint_load(os.path.join(GOLD, f"ref_ckpt_{run}.pylo"),
                                                   mode=mode)
    for step in (3, 4):
        for j, p in enumerate(params):
            p.grad = torch.from_numpy(z[f"{run}/step{step}/grad{j}"]).cuda()
        opt.step()
        torch.cuda.synchronize()
        for j, p in enumerate(params):
            got = p.detach().cpu().numpy()
            want = z[f"{run}/step{step}/param{j}"]
            if mode == "strict":
                assert got.tobytes() == want.tobytes(), (step, j)
            else:
                assert np.max(np.abs(got - want) / (1 + np.abs(want))) <= 1e-5, (step, j)
    for j, p in enumerate(params):
        quad = opt.state[p]["quad"].cpu().numpy()
        assert quad[:, 3].tobytes() == z[f"{run}/final/state{j}/V"].reshape(-1).tobytes()
        assert quad[:, 2].tobytes() == z[f"{run}/final/state{j}/M2"].reshape(-1).tobytes()
        assert opt.state[p]["row_factors"].cpu().numpy()[1].tobytes() == \
            z[f"{run}/final/state{j}/r1"].tobytes()
    assert opt.T == 5


def test_checkpoint_roundtrip_after_gpu_steps(tmp_path):
    """GPU optimizer -> checkpoint -> fresh optimizer: identical next step."""
    import torch

    import paper_2506_10315_b200 as P
    from paper_2506_10315_b200 import container

    rng = np.random.default_rng(3)
    shapes = [(64, 96), (64,), (10, 64)]
    a = [torch.nn.Parameter(torch.from_numpy((rng.standard_normal(s) * 0.05).astype(np.float32)).cuda())
         for s in shapes]
    opt = P.LearnedOptimizer(a, weight_decay=0.02, mode="strict")
    gs = [[(rng.standard_normal(s) * 1e-2).astype(np.float32) for s in shapes] for _ in range(3)]
    for k in range(2):
        for p, g in zip(a, gs[k]):
            p.grad = torch.from_numpy(g).cuda()
        opt.step()
    container.checkpoint_save(opt, tmp_path / "c.pylo")
    opt2, b, _ = container.checkpoint_load(tmp_path / "c.pylo", mode="strict")
    for p, g in zip(a, gs[2]):
        p.grad = torch.from_numpy(g).cuda()
    for p, g in zip(b, gs[2]):
        p.grad = torch.from_numpy(g.reshape(p.shape)).cuda()
    opt.step()
    opt2.step()
    for p, q in zip(a, b):
        assert p.detach().cpu().numpy().reshape(-1).tobytes() == q.detach().cpu().numpy().reshape(-1).tobytes()
