"""Golden vectors for the reference's baseline optimizers (adam_step,
adafactor_step, pkg/src/lopt/optim.py:187-217), produced by running the
REFERENCE in this container (it does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \\
        python tests/golden/gen_baselines.py

-> tests/golden/baseline_cases.npz.  Checked bitwise against the oracle by
tests/test_oracle_golden.py and against the GPU by tests/test_gpu_baselines.py.
"""

from __future__ import annotations

import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gen_golden import OUT, _import_reference  # noqa: E402

F32 = np.float32
ADAM_SHAPES = [(3, 3), (17, 33), (1, 1), (257, 5)]
FACTOR_SHAPES = [(5, 7), (64, 33), (1, 10), (10, 1), (130, 70)]


def main():
    _, _, optim, _ = _import_reference()
    out = {}
    rng = np.random.default_rng(41)
    for k, s in enumerate(ADAM_SHAPES):
        th = rng.standard_normal(s, dtype=F32)
        m = np.zeros(s, F32)
        v = np.zeros(s, F32)
        out[f"adam{k}/theta0"] = th
        for t in range(1, 5):
            g = (rng.standard_normal(s, dtype=F32) * F32(0.1 * t)).astype(F32)
            out[f"adam{k}/g{t}"] = g
            lr = 1e-3 if t != 3 else 0.05
            th, m, v = optim.adam_step(th, g, m, v, lr=lr, t=t)
            out[f"adam{k}/theta{t}"] = th
            out[f"adam{k}/m{t}"] = m
            out[f"adam{k}/v{t}"] = v
    for k, s in enumerate(FACTOR_SHAPES):
        th = rng.standard_normal(s, dtype=F32)
        r = np.zeros(s[0], F32)
        c = np.zeros(s[1], F32)
        out[f"afac{k}/theta0"] = th
        for t in range(1, 4):
            g = (rng.standard_normal(s, dtype=F32) * F32(0.05)).astype(F32)
            out[f"afac{k}/g{t}"] = g
            th, r, c = optim.adafactor_step(th, g, r, c, lr=1e-2 if t == 2 else 1e-3)
            out[f"afac{k}/theta{t}"] = th
            out[f"afac{k}/r{t}"] = r
            out[f"afac{k}/c{t}"] = c
    np.savez_compressed(os.path.join(OUT, "baseline_cases.npz"), **out)
    print("wrote", len(out), "arrays")


if __name__ == "__main__":
    main()
