"""Known-answer tests of the tcgen05 building blocks (descriptors, TMEM
layouts, commit/mbarrier) against a float64 matmul.  Needs a B200."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["bf16", "fp16"])
@pytest.mark.parametrize("a_in_tmem", [0, 1])
@pytest.mark.parametrize("K", [16, 32, 64])
def test_umma_known_answer(a_in_tmem, K, dtype):
    import torch

    from paper_2506_10315_b200 import _lib

    L = _lib.require_cuda()
    g = torch.Generator().manual_seed(K + 7 * a_in_tmem)
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float16
    A = torch.randn(128, K, generator=g).to(tdt)
    B = torch.randn(32, K, generator=g).to(tdt)
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.empty(128, 32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    flags = a_in_tmem | (2 if dtype == "fp16" else 0)
    _lib.check(L.lopt_selftest_umma(flags, K, Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), s))
    torch.cuda.synchronize()
    want = A.double() @ B.double().T
    np.testing.assert_allclose(D.cpu().double().numpy(), want.numpy(), rtol=1e-5, atol=1e-5)
