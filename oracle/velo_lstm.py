"""numpy restatement of the VeLO per-tensor hypernetwork of this build.

TEST INFRASTRUCTURE ONLY (see oracle/oracle.py).

The reference has no VeLO LSTM (SPEC.md:14 lists it out of scope; the
reference's "VeLO" is the 29-column VELO_MLP feature set with one global MLP,
features.py:24-28).  The north star asks for "a per-tensor LSTM hypernetwork
that mixes a bank of per-parameter MLPs", so the build defines one
 and pins its CUDA kernel
(paper_2506_10315_b200/csrc/lopt_velo.cu) against this file.  PARITY
UNPINNED against any external reference: there is no released VeLO weight set
or reference implementation here to compare with.

Definition, per tensor j and step:
    x   = [f32(log(sumsq_k / count + 1e-5)) for the 29 VELO_MLP columns,
           tanh(f32(t) / x) for the 11 TIME_XS horizons (features.py:52),
           log(max(loss, 1e-8)), its EMA (0.9 decay)]            (42 inputs)
    g   = b + W_x x + W_h h           sequential f32 fma, x first then h
    c'  = sig(g_f) c + sig(g_i) tanh(g_g),   h' = sig(g_o) tanh(c')
    a   = softmax(b_o + W_o h')        (K bank weights)
    W_j = sum_k a_k bank_k             (packed MLP, every entry, fma over k)
"""

from __future__ import annotations

import math

import numpy as np

F32 = np.float32
N_IN = 42
TIME_XS = (1.0, 3.0, 10.0, 30.0, 100.0, 300.0, 1000.0, 3000.0, 1e4, 3e4, 1e5)


def hyper_layout(H: int, K: int) -> dict:
    sizes = {"Wx": 4 * H * N_IN, "Wh": 4 * H * H, "b": 4 * H, "Wo": K * H, "bo": K}
    out, off = {}, 0
    for k, s in sizes.items():
        out[k] = (off, s)
        off += s
    out["total"] = off
    return out


def random_hyper(H=16, K=4, seed=0, scale=0.1):
    """Seeded random hypernetwork parameters (the build's random init)."""
    rng = np.random.default_rng(seed)
    lay = hyper_layout(H, K)
    p = (rng.standard_normal(lay["total"]) * scale).astype(F32)
    # forget-gate bias of +1, the usual LSTM initialisation
    off, _ = lay["b"]
    p[off + H: off + 2 * H] = F32(1.0)
    return p


def random_bank(K=4, d_feat=29, hidden=(32, 32), seed=0, scale=0.2):
    """K per-element MLPs, each drawn like engine.py:178-192 random_weights."""
    from oracle.oracle import random_weights

    mats = []
    for k in range(K):
        w = random_weights(d_feat, hidden=hidden, seed=seed * 1000 + k, scale=scale)
        mats.append(np.concatenate([a.ravel() for wb in w.layers for a in wb]).astype(F32))
    return np.stack(mats)


def loss_features(loss, ema):
    """Host scalars: (log loss, EMA of log loss); ema None on the first step."""
    lv = math.log(max(float(loss), 1e-8))
    ema = lv if ema is None else 0.9 * ema + 0.1 * lv
    return np.array([lv, ema], F32), ema


def _fma_chain(start, ws, xs):
    acc = np.float32(start)
    for w, x in zip(ws, xs):
        acc = np.float32(math.fma(float(w), float(x), float(acc))) if hasattr(math, "fma") else \
            np.float32(np.float64(w) * np.float64(x) + np.float64(acc))
    return acc


def _sig(z):
    return F32(1.0) / (F32(1.0) + np.exp(-F32(z)))


def velo_mix(hyper, lstm_state, bank, sumsq, counts, t, loss_feats, H=16, K=4):
    """One hypernetwork step for every tensor.  sumsq: (count, 29) f64,
    counts: (count,), lstm_state: (count, 2H) f32 (updated copy returned).
    Returns (per-tensor packed MLPs (count, stride), mixing weights, new state)."""
    lay = hyper_layout(H, K)
    get = lambda k: hyper[lay[k][0]: lay[k][0] + lay[k][1]]
    Wx = get("Wx").reshape(4 * H, N_IN)
    Wh = get("Wh").reshape(4 * H, H)
    bg = get("b")
    Wo = get("Wo").reshape(K, H)
    bo = get("bo")
    tf = np.tanh(F32(t) / np.array(TIME_XS, dtype=F32)).astype(F32)
    new_state = lstm_state.copy()
    mixed, alphas = [], []
    for j in range(sumsq.shape[0]):
        x = np.zeros(N_IN, F32)
        x[:29] = np.log(sumsq[j] / float(counts[j]) + 1e-5).astype(F32)
        x[29:40] = tf
        x[40:42] = loss_feats
        h = lstm_state[j, :H].astype(F32)
        c = lstm_state[j, H:].astype(F32)
        xin = np.concatenate([x, h])
        W = np.concatenate([Wx, Wh], axis=1)
        g = np.array([_fma_chain(bg[q], W[q], xin) for q in range(4 * H)], F32)
        ig, fg = _sig(g[:H]), _sig(g[H:2 * H])
        gg, og = np.tanh(g[2 * H:3 * H]).astype(F32), _sig(g[3 * H:])
        cn = (fg * c + ig * gg).astype(F32)
        hn = (og * np.tanh(cn)).astype(F32)
        new_state[j, :H] = hn
        new_state[j, H:] = cn
        logits = np.array([_fma_chain(bo[k], Wo[k], hn) for k in range(K)], F32)
        e = np.exp(logits - logits.max()).astype(F32)
        a = (e / e.sum(dtype=F32)).astype(F32)
        alphas.append(a)
        mixed.append((a.astype(np.float64)[:, None] * bank.astype(np.float64)).sum(0).astype(F32))
    return np.stack(mixed), np.stack(alphas), new_state
