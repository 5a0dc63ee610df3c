"""Pin the C oracle against fixtures produced by the reference itself
(tests/golden/gen_golden.py), bit for bit, plus the reference's own
known-answer tests restated."""

import math

import numpy as np
import pytest

from conftest import F32, load_golden

ENGINE_SHAPES = [(1, 1), (1, 130), (130, 1), (5, 64), (7, 63), (3, 65), (33, 70), (64, 64),
                 (17, 129)]
MODEL_SHAPES = [(16, 98), (16, 1), (10, 16), (10, 1)]


def _state_from(O, G, key, m, n):
    s = O.OState.zeros(m, n)
    for i in range(3):
        s.M[i] = G[f"{key}/M{i}"]
        s.r[i] = G[f"{key}/r{i}"]
        s.c[i] = G[f"{key}/c{i}"]
    s.V = G[f"{key}/V"]
    if f"{key}/t" in G:
        s.t = int(G[f"{key}/t"][0])
    return s


def _bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and a.tobytes() == b.tobytes()


# ---------------------------------------------------------------------------
# accumulators: numpy reduction orders reproduced exactly


@pytest.mark.parametrize("shape", [(3, 4), (9000, 1), (2, 9000), (300, 2), (257, 129), (1, 1)])
def test_state_step_matches_reference_bitwise(oracle, shape):
    O = oracle
    G = load_golden("state_cases.npz")
    m, n = shape
    key = f"state/{m}x{n}"
    s = O.OState.zeros(m, n)
    for k in range(2):
        s = O.state_step(s, G[f"{key}/g{k}"])
    for i in range(3):
        assert _bits_equal(s.M[i], G[f"{key}/M{i}"])
        assert _bits_equal(s.r[i], G[f"{key}/r{i}"])
        assert _bits_equal(s.c[i], G[f"{key}/c{i}"])
    assert _bits_equal(s.V, G[f"{key}/V"])
    assert _bits_equal(np.array(O.factor_means(s), F32), G[f"{key}/mr"])


# reference KATs, pkg/tests/test_state.py:118-185


def test_adafactor_hand_means(oracle):
    O = oracle
    g = np.array([[1.0, 2.0], [3.0, 4.0]], F32)
    s = O.state_step(O.OState.zeros(2, 2), g, betas=(0, 0, 0, 0, 0, 0, 0))
    assert np.array_equal(s.r[0], np.array([2.5, 12.5], F32))
    assert np.array_equal(s.c[0], np.array([5.0, 10.0], F32))
    assert np.array_equal(s.M[0], g) and np.array_equal(s.V, g * g)


def test_state_step_twice_constant_gradient(oracle):
    O = oracle
    s = O.OState.zeros(1, 1)
    g = np.ones((1, 1), F32)
    betas = (0.9, 0.9, 0.9, 0.999, 0.9, 0.99, 0.999)
    s = O.state_step(O.state_step(s, g, betas), g, betas)
    b = F32(0.9)
    omb = F32(1.0) - b
    assert s.M[0][0, 0] == b * (b * F32(0.0) + omb * F32(1.0)) + omb * F32(1.0)
    assert abs(float(s.M[0][0, 0]) - 0.19) < 1e-6 and s.t == 2


def test_state_step_rejects_nonfinite(oracle):
    O = oracle
    bad = np.ones((2, 2), F32)
    bad[1, 1] = np.nan
    with pytest.raises(O.OracleError):
        O.state_step(O.OState.zeros(2, 2), bad)


# ---------------------------------------------------------------------------
# engine: features, pass-1 sums, pass-2 outputs


@pytest.mark.parametrize("spec_name", ["small_fc_lopt", "velo_mlp"])
@pytest.mark.parametrize("shape", ENGINE_SHAPES)
def test_engine_matches_reference_bitwise(oracle, spec_name, shape):
    O = oracle
    G = load_golden("engine_cases.npz")
    m, n = shape
    key = f"{spec_name}/{m}x{n}"
    kind = O.KIND_BY_NAME[spec_name]
    s = _state_from(O, G, key, m, n)
    W, g = G[key + "/W"], G[key + "/g"]
    for row, idx in zip(G[key + "/feat"], G[key + "/idx"]):
        assert _bits_equal(O.features_at(int(idx), W, g, s, kind), row)
    for workers in (1, 3):
        sumsq, count = O.fused_stats(W, g, s, kind, workers=workers)
        assert count == m * n
        assert _bits_equal(sumsq, G[key + f"/sumsq_w{workers}"])
    w = O.random_weights(39 if kind == O.SMALL_FC_LOPT else 29, seed=int(G[key + "/wseed"][0]))
    for lr in (1.0, 0.3):
        out, maxabs, _ = O.step_fused(W, g, s, w, kind, lr=lr)
        assert _bits_equal(out, G[key + f"/out_lr{lr}"])
        assert maxabs == pytest.approx(float(G[key + f"/maxabs_lr{lr}"][0]), rel=0, abs=0)


def test_zero_network_is_bitwise_noop(oracle):
    """pkg/tests/test_engine.py:249-259 restated on the oracle."""
    O = oracle
    rng = np.random.default_rng(1)
    m, n = 33, 70
    s = O.OState.zeros(m, n)
    for _ in range(2):
        s = O.state_step(s, rng.standard_normal((m, n)).astype(F32))
    g = rng.standard_normal((m, n)).astype(F32)
    W = rng.standard_normal((m, n)).astype(F32)
    W[0, 0] = -0.0
    W[0, 1] = 0.0
    out, _, _ = O.step_fused(W, g, s, O.zero_weights(39), O.SMALL_FC_LOPT)
    assert out.tobytes() == W.tobytes()


def test_apply_update_kats(oracle):
    """test_engine.py:86-95: a selector net gives dir=1, mag in {0, 1}."""
    O = oracle
    # one-element tensor, zero layers except the output biases
    w = O.zero_weights(39)
    (w3, b3) = w.layers[2]
    b3[:] = [1.0, 0.0]
    s = O.state_step(O.OState.zeros(1, 1), np.ones((1, 1), F32))
    out, _, _ = O.step_fused(np.zeros((1, 1), F32), np.ones((1, 1), F32), s, w, O.SMALL_FC_LOPT)
    assert abs(float(out[0, 0]) - (-0.01)) < 1e-9
    b3[:] = [1.0, 1.0]
    out, _, _ = O.step_fused(np.zeros((1, 1), F32), np.ones((1, 1), F32), s, w, O.SMALL_FC_LOPT)
    assert abs(float(out[0, 0]) - (-0.01 * math.exp(0.01))) < 1e-9
    assert round(float(out[0, 0]), 7) == -0.0101005


# ---------------------------------------------------------------------------
# facade: multi-step opt_step with schedules and decay


@pytest.mark.parametrize("run", ["small_const", "velo_cos_wd"])
def test_opt_step_trajectory_matches_reference_bitwise(oracle, run):
    O = oracle
    G = load_golden("optstep_cases.npz")
    cfg = {
        "small_const": dict(kind=O.SMALL_FC_LOPT, sched=("constant", 1.0, 0.0, 0, 1), wd=0.0, wseed=0),
        "velo_cos_wd": dict(kind=O.VELO_MLP, sched=("cosine", 0.8, 0.05, 2, 8), wd=0.01, wseed=1),
    }[run]
    params = [G[f"{run}/init/param{j}"].reshape(O.view_2d(s)).copy() for j, s in enumerate(MODEL_SHAPES)]
    states = [O.OState.zeros(*p.shape) for p in params]
    w = O.random_weights(39 if cfg["kind"] == O.SMALL_FC_LOPT else 29, seed=cfg["wseed"])
    grng = np.random.default_rng(78)
    for step in range(6):
        grads = [(grng.standard_normal(p.shape) * 1e-2).astype(F32) for p in params]
        lr = O.schedule_lr(*cfg["sched"], step)
        O.opt_step(params, states, grads, w, cfg["kind"], lr, weight_decay=cfg["wd"], threads=2)
        for j, p in enumerate(params):
            assert _bits_equal(p, G[f"{run}/step{step}/param{j}"].reshape(p.shape)), (step, j)
    for j, s in enumerate(states):
        for i in range(3):
            assert _bits_equal(s.M[i], G[f"{run}/final/state{j}/M{i}"].reshape(s.M[i].shape))
            assert _bits_equal(s.r[i], G[f"{run}/final/state{j}/r{i}"])
            assert _bits_equal(s.c[i], G[f"{run}/final/state{j}/c{i}"])


def test_schedule_matches_reference_kats(oracle):
    """pkg/tests/test_optim.py:34-75."""
    O = oracle
    assert O.schedule_lr("cosine", 0.5, 0.01, 10, 100, 10) == 0.5
    assert O.schedule_lr("cosine", 0.5, 0.01, 10, 100, 100) == 0.01
    assert O.schedule_lr("cosine", 0.5, 0.01, 10, 100, 0) == 0.0
    assert O.schedule_lr("cosine", 0.5, 0.01, 10, 100, 5) == 0.5 * (5 / 10)
    assert O.schedule_lr("cosine", 1.0, 0.2, 0, 8, 4) == pytest.approx(0.6, rel=1e-12)


def test_view_rule():
    from oracle.oracle import view_2d

    assert view_2d(()) == (1, 1)
    assert view_2d((5,)) == (5, 1)
    assert view_2d((1, 768)) == (1, 768)
    assert view_2d((1, 1, 768)) == (1, 768)
    assert view_2d((1, 197, 768)) == (197, 768)
    assert view_2d((768, 3, 16, 16)) == (768, 768)


BASE = load_golden("baseline_cases.npz")


@pytest.mark.parametrize("k", range(4))
def test_adam_oracle_bitwise(oracle, k):
    """Oracle adam_step == the reference's (optim.py:187-198), 4 chained steps."""
    th = BASE[f"adam{k}/theta0"]
    m = np.zeros_like(th)
    v = np.zeros_like(th)
    for t in range(1, 5):
        th, m, v = oracle.adam_step(th, BASE[f"adam{k}/g{t}"], m, v, lr=1e-3 if t != 3 else 0.05, t=t)
        for nm, got in (("theta", th), ("m", m), ("v", v)):
            assert np.array_equal(got.view(np.uint32), BASE[f"adam{k}/{nm}{t}"].view(np.uint32)), (nm, t)


@pytest.mark.parametrize("k", range(5))
def test_adafactor_oracle_bitwise(oracle, k):
    """Oracle adafactor_step == the reference's (optim.py:201-217), 3 chained steps."""
    th = BASE[f"afac{k}/theta0"]
    r = np.zeros(th.shape[0], np.float32)
    c = np.zeros(th.shape[1], np.float32)
    for t in range(1, 4):
        th, r, c = oracle.adafactor_step(th, BASE[f"afac{k}/g{t}"], r, c, lr=1e-2 if t == 2 else 1e-3)
        for nm, got in (("theta", th), ("r", r), ("c", c)):
            assert np.array_equal(got.view(np.uint32), BASE[f"afac{k}/{nm}{t}"].view(np.uint32)), (nm, t)


def test_adam_oracle_rejects_t0(oracle):
    with pytest.raises(ValueError):
        oracle.adam_step(np.zeros(2, np.float32), np.zeros(2, np.float32), np.zeros(2, np.float32),
                    np.zeros(2, np.float32), t=0)
