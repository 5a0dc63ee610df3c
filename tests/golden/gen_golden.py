"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box):

    PYTHONDONTWRITEBYTECODE=1 NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/gen_golden.py

Outputs tests/golden/*.npz and the reference-written PYLO files
tests/golden/ref_*.pylo (container / checkpoint interop).  Every array in them is produced by the
reference's own public functions (pkg/src/lopt/...), on inputs generated here
from fixed seeds.  tests/test_oracle_golden.py checks the C oracle against
these files bit for bit; the GPU parity tests then check the CUDA path
against the oracle.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF_SRC = os.environ.get("LOPT_REFERENCE_SRC", "/root/reference/pkg/src")
OUT = os.path.dirname(os.path.abspath(__file__))
F32 = np.float32


def _import_reference():
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache")
    sys.dont_write_bytecode = True
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import lopt  # noqa: F401
    from lopt import engine, features, optim, state
    return engine, features, optim, state


def advanced_state(state_mod, rng, m, n, steps=2, betas=None, grad_scale=1.0):
    """pkg/tests/conftest.py:31-43, restated (same generator calls)."""
    betas = betas or state_mod.BetaConfig()
    s = state_mod.OptState.zeros(m, n)
    g = np.zeros((m, n), dtype=F32)
    for _ in range(steps):
        g = (rng.standard_normal((m, n)) * grad_scale).astype(F32)
        s = state_mod.state_step(s, g, betas)
    return s, g


ENGINE_SHAPES = [(1, 1), (1, 130), (130, 1), (5, 64), (7, 63), (3, 65), (33, 70), (64, 64),
                 (17, 129)]


def engine_cases(engine, features, state_mod):
    """Per-tensor engine outputs: features at sampled indices, pass-1 sums for
    several worker counts, and step_fused / step_naive at lr 1 and lr 0.3."""
    out = {}
    for spec_name in ("small_fc_lopt", "velo_mlp"):
        spec = features.spec_by_name(spec_name)
        for ci, (m, n) in enumerate(ENGINE_SHAPES):
            key = f"{spec_name}/{m}x{n}"
            rng = np.random.default_rng(1000 + 17 * ci + (0 if spec_name == "small_fc_lopt" else 7))
            s, g = advanced_state(state_mod, rng, m, n, steps=1 + ci % 3, grad_scale=10.0 ** (ci % 3 - 1))
            W = rng.standard_normal((m, n)).astype(F32)
            w = engine.random_weights(spec.d_feat, seed=ci)
            idxs = np.unique(rng.integers(0, m * n, size=min(8, m * n)))
            feats = np.stack([features.construct_features_at(int(i), W, g, s, spec) for i in idxs])
            out[key + "/W"] = W
            out[key + "/g"] = g
            for i in range(3):
                out[key + f"/M{i}"] = s.M[i]
                out[key + f"/r{i}"] = s.r[i]
                out[key + f"/c{i}"] = s.c[i]
            out[key + "/V"] = s.V
            out[key + "/t"] = np.array([s.t], np.int64)
            out[key + "/wseed"] = np.array([ci], np.int64)
            out[key + "/idx"] = idxs.astype(np.int64)
            out[key + "/feat"] = feats
            for workers in (1, 3):
                st = engine.fused_stats(W, g, s, spec, workers=workers)
                out[key + f"/sumsq_w{workers}"] = st.sumsq
            for lr in (1.0, 0.3):
                p2, rep = engine.step_fused(W, g, s, w, spec, lr=lr)
                out[key + f"/out_lr{lr}"] = p2.data
                out[key + f"/maxabs_lr{lr}"] = np.array([rep.max_abs_update], np.float64)
                # the naive class (engine.py:751-826): BLAS MLP, cross-path tolerance
                p3, _ = engine.step_naive(W, g, s, w, spec, lr=lr)
                out[key + f"/naive_lr{lr}"] = p3.data
    return out


# A small MNIST-shaped MLP (the survey's C1 uses 784->128->10; this is the
# same topology at 1/8 width so the fixture stays small).
MODEL_SHAPES = [(16, 98), (16, 1), (10, 16), (10, 1)]


def optstep_cases(engine, features, optim, state_mod):
    out = {}
    runs = {
        "small_const": dict(spec="small_fc_lopt", sched=optim.ScheduleConfig(kind="constant", max_lr=1.0),
                            wd=0.0, steps=6, wseed=0),
        "velo_cos_wd": dict(spec="velo_mlp",
                            sched=optim.ScheduleConfig(kind="cosine", max_lr=0.8, min_lr=0.05,
                                                       warmup_steps=2, total_steps=8),
                            wd=0.01, steps=6, wseed=1),
    }
    for name, cfg in runs.items():
        spec = features.spec_by_name(cfg["spec"])
        rng = np.random.default_rng(77)
        named = [(f"t{i}", (rng.standard_normal(s) * 0.05).astype(F32)) for i, s in enumerate(MODEL_SHAPES)]
        w = engine.random_weights(spec.d_feat, seed=cfg["wseed"])
        h = optim.OptimizerHandle.fresh(named, w, spec, schedule=cfg["sched"], weight_decay=cfg["wd"])
        grng = np.random.default_rng(78)
        for step in range(cfg["steps"]):
            grads = [(grng.standard_normal(p.shape) * 1e-2).astype(F32) for _, p in h.params]
            optim.opt_step(h, grads)
            for j, (tn, p) in enumerate(h.params):
                out[f"{name}/step{step}/param{j}"] = p.data
        for j, s in enumerate(h.states):
            for i in range(3):
                out[f"{name}/final/state{j}/M{i}"] = s.M[i]
                out[f"{name}/final/state{j}/r{i}"] = s.r[i]
                out[f"{name}/final/state{j}/c{i}"] = s.c[i]
            out[f"{name}/final/state{j}/V"] = s.V
        for j, (_, p0) in enumerate(named):
            out[f"{name}/init/param{j}"] = p0
    return out


def state_cases(state_mod, features):
    """Accumulator + factor-mean outputs on shapes that exercise numpy's
    reduction orders (long rows -> pairwise; (m,1) -> pairwise over axis 0;
    > 8192 rows -> buffered f64 cast)."""
    out = {}
    rng = np.random.default_rng(5)
    for m, n in [(3, 4), (9000, 1), (2, 9000), (300, 2), (257, 129), (1, 1)]:
        key = f"state/{m}x{n}"
        s = state_mod.OptState.zeros(m, n)
        gs = []
        for k in range(2):
            g = (rng.standard_normal((m, n)) * (1.0 + k)).astype(F32)
            gs.append(g)
            s = state_mod.state_step(s, g, state_mod.BetaConfig())
        for k, g in enumerate(gs):
            out[key + f"/g{k}"] = g
        for i in range(3):
            out[key + f"/M{i}"] = s.M[i]
            out[key + f"/r{i}"] = s.r[i]
            out[key + f"/c{i}"] = s.c[i]
        out[key + "/V"] = s.V
        out[key + "/mr"] = np.array(features.factor_means(s), F32)
    return out


def ckpt_cases(engine, features, optim, state_mod):
    """Reference-written PYLO files (weights + checkpoints after 3 steps) and
    the reference's continuation for 2 more steps from each checkpoint."""
    from lopt import tensors

    out = {}
    runs = {
        "small_const": dict(spec="small_fc_lopt", sched=optim.ScheduleConfig(kind="constant", max_lr=0.7),
                            wd=0.0, wseed=3),
        "velo_cos_wd": dict(spec="velo_mlp",
                            sched=optim.ScheduleConfig(kind="cosine", max_lr=0.8, min_lr=0.05,
                                                       warmup_steps=2, total_steps=8),
                            wd=0.01, wseed=4),
    }
    for name, cfg in runs.items():
        spec = features.spec_by_name(cfg["spec"])
        rng = np.random.default_rng(91)
        named = [(f"layer{i}", (rng.standard_normal(s) * 0.05).astype(F32))
                 for i, s in enumerate(MODEL_SHAPES)]
        w = engine.random_weights(spec.d_feat, seed=cfg["wseed"])
        engine.save_weights(w, spec, os.path.join(OUT, f"ref_weights_{name}.pylo"))
        h = optim.OptimizerHandle.fresh(named, w, spec, schedule=cfg["sched"], weight_decay=cfg["wd"])
        grng = np.random.default_rng(92)
        for step in range(5):
            if step == 3:
                optim.checkpoint_save(h, os.path.join(OUT, f"ref_ckpt_{name}.pylo"))
            grads = [(grng.standard_normal(p.shape) * 1e-2).astype(F32) for _, p in h.params]
            optim.opt_step(h, grads)
            if step >= 3:
                for j, g in enumerate(grads):
                    out[f"{name}/step{step}/grad{j}"] = g
                for j, (_, p) in enumerate(h.params):
                    out[f"{name}/step{step}/param{j}"] = p.data
        for j, s in enumerate(h.states):
            out[f"{name}/final/state{j}/V"] = s.V
            out[f"{name}/final/state{j}/M2"] = s.M[2]
            out[f"{name}/final/state{j}/r1"] = s.r[1]
    # a container with every dtype and a 0-d and an empty array, for the
    # byte-for-byte writer comparison
    tensors.file_save({"a": np.arange(6, dtype=F32).reshape(2, 3), "b": np.array(3.5),
                       "c": np.arange(5, dtype=np.int64), "d": np.zeros((0, 4), F32)},
                      {"kind": "misc", "note": "unicode \u00e9"}, os.path.join(OUT, "ref_misc.pylo"))
    return out


def main():
    engine, features, optim, state_mod = _import_reference()
    np.savez_compressed(os.path.join(OUT, "ckpt_cases.npz"),
                        **ckpt_cases(engine, features, optim, state_mod))
    np.savez_compressed(os.path.join(OUT, "engine_cases.npz"), **engine_cases(engine, features, state_mod))
    np.savez_compressed(os.path.join(OUT, "optstep_cases.npz"),
                        **optstep_cases(engine, features, optim, state_mod))
    np.savez_compressed(os.path.join(OUT, "state_cases.npz"), **state_cases(state_mod, features))
    for f in sorted(os.listdir(OUT)):
        if f.endswith((".npz", ".pylo")):
            print(f, os.path.getsize(os.path.join(OUT, f)))


if __name__ == "__main__":
    main()
