"""The exponential of the strict path: glibc's expf algorithm restated in
double arithmetic (paper_2506_10315_b200/csrc/lopt_common.cuh glibc_expf).
numba's np.exp on float32 is glibc expf (pkg/src/lopt/engine.py:537), so the
restatement must equal the host libm bit for bit."""

import os
import subprocess

import numpy as np
import pytest

from conftest import ROOT


def test_restated_expf_equals_libm_on_strided_inputs(oracle):
    exe = os.path.join(ROOT, "oracle", "_build", "expf_check")
    if not os.path.exists(exe):
        oracle.build()
    # every 7th float bit pattern (~6e8 inputs); stride 1 = all 2^32
    out = subprocess.run([exe, "7"], capture_output=True, text=True, check=True).stdout.split()
    mism, tot = int(out[0]), int(out[1])
    assert tot > 600_000_000 and mism == 0


@pytest.mark.gpu
def test_device_expf_equals_libm(oracle):
    import torch

    from paper_2506_10315_b200 import _lib

    L = _lib.require_cuda()
    rng = np.random.default_rng(0)
    xs = [rng.standard_normal(2_000_000).astype(np.float32) * s for s in (0.01, 1.0, 30.0)]
    xs.append(rng.integers(0, 2**32, 4_000_000, dtype=np.uint64).astype(np.uint32).view(np.float32))
    x = np.concatenate(xs)
    x = x[~np.isnan(x)]
    xd = torch.from_numpy(x).cuda()
    yd = torch.empty_like(xd)
    _lib.check(L.lopt_selftest_expf(xd.data_ptr(), yd.data_ptr(), x.size,
                                    torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    want = oracle.libm_expf(x)
    got = yd.cpu().numpy()
    assert np.count_nonzero(got.view(np.uint32) != want.view(np.uint32)) == 0
