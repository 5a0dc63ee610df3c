"""Shared test setup.

Markers: `gpu` tests need a B200 (run with `-m gpu` on the GPU box); everything
else runs on CPU in the build container.
"""

import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
F32 = np.float32


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def advanced_state(rng, m, n, steps=2, grad_scale=1.0):
    """Same generator calls as the reference's conftest.advanced_state
    (pkg/tests/conftest.py:31-43), built on the oracle."""
    from oracle import oracle as O

    s = O.OState.zeros(m, n)
    g = np.zeros((m, n), dtype=F32)
    for _ in range(steps):
        g = (rng.standard_normal((m, n)) * grad_scale).astype(F32)
        s = O.state_step(s, g)
    return s, g


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O

    O.lib()
    return O
