"""Known-answer tests of the tcgen05 building blocks (descriptors, TMEM
layouts, commit/mbarrier) against a float64 matmul.  Needs a B200."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("a_in_tmem", [0, 1])
@pytest.mark.parametrize("K", [16, 32, 64])
def test_umma_bf16_known_answer(a_in_tmem, K):
    import torch

    from paper_2506_10315_b200 import _lib

    L = _lib.require_cuda()
    g = torch.Generator().manual_seed(K + 7 * a_in_tmem)
    A = torch.randn(128, K, generator=g).to(torch.bfloat16)
    B = torch.randn(32, K, generator=g).to(torch.bfloat16)
    Ad, Bd = A.cuda(), B.cuda()
    D = torch.empty(128, 32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    _lib.check(L.lopt_selftest_umma(a_in_tmem, K, Ad.data_ptr(), Bd.data_ptr(), D.data_ptr(), s))
    torch.cuda.synchronize()
    want = A.double() @ B.double().T
    np.testing.assert_allclose(D.cpu().double().numpy(), want.numpy(), rtol=1e-5, atol=1e-5)
