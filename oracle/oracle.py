"""numpy/ctypes front end of the CPU oracle (oracle/lopt_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / `--impl reference` legs as the checker.  The product
package (paper_2506_10315_b200) never imports this module.

The functions mirror the reference API (paths relative to the reference repo):

    state_step          pkg/src/lopt/state.py:116-130
    time_features       pkg/src/lopt/features.py:125-130  (numpy, same call)
    factor_means        pkg/src/lopt/features.py:133-135
    normalization_scale pkg/src/lopt/features.py:138-140
    features_at         pkg/src/lopt/features.py:304-315
    fused_stats         pkg/src/lopt/engine.py:619-654
    fused_apply         pkg/src/lopt/engine.py:657-710
    step_fused          pkg/src/lopt/engine.py:713-748
    opt_step            pkg/src/lopt/optim.py:144-180 (multi-tensor, OpenMP)
    random_weights      pkg/src/lopt/engine.py:178-192
    schedule_lr         pkg/src/lopt/optim.py:69-89
    adam_step           pkg/src/lopt/optim.py:187-198  (numpy, f32 op by op)
    adafactor_step      pkg/src/lopt/optim.py:201-217  (numpy, f32 op by op)

Parity of this oracle with the reference is pinned by tests/test_oracle_golden.py
against fixtures generated from the reference itself (tests/golden/).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

F32 = np.float32
SMALL_FC_LOPT = 0
VELO_MLP = 1
KIND_BY_NAME = {"small_fc_lopt": SMALL_FC_LOPT, "velo_mlp": VELO_MLP}
TIME_XS = (1.0, 3.0, 10.0, 30.0, 100.0, 300.0, 1000.0, 3000.0, 1e4, 3e4, 1e5)
DEFAULT_BETAS = (0.1, 0.5, 0.9, 0.999, 0.9, 0.99, 0.999)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "_build", "liblopt_oracle.so")

OK, ERR_NONFINITE_GRAD, ERR_OVERFLOW, ERR_SHAPE, ERR_ALLOC = 0, 1, 2, 3, 4


class OracleError(RuntimeError):
    def __init__(self, code: int, index: int = -1):
        self.code = code
        self.index = index
        super().__init__(f"oracle status {code} (tensor {index})")


def build() -> str:
    """Compile the oracle with its Makefile (gcc, seconds)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _SO


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(
            os.path.join(_HERE, "lopt_oracle.c")
        ):
            build()
        L = ctypes.CDLL(_SO)
        fp = ctypes.POINTER(ctypes.c_float)
        dp = ctypes.POINTER(ctypes.c_double)
        i64 = ctypes.c_int64
        L.lo_state_step.argtypes = [i64, i64, fp] + [fp] * 10 + [dp]
        L.lo_state_step.restype = ctypes.c_int
        L.lo_factor_mean.argtypes = [fp, i64]
        L.lo_factor_mean.restype = ctypes.c_float
        L.lo_features_at.argtypes = [ctypes.c_int, i64, i64, fp, fp] + [fp] * 10 + [fp, i64, fp]
        L.lo_features_at.restype = None
        L.lo_fused_stats.argtypes = (
            [ctypes.c_int, i64, i64, fp, fp] + [fp] * 10 + [fp, i64, i64, i64, dp]
        )
        L.lo_fused_stats.restype = ctypes.c_int
        L.lo_normalization_scale.argtypes = [ctypes.c_int, dp, i64, fp]
        L.lo_normalization_scale.restype = None
        L.lo_fused_apply.argtypes = (
            [ctypes.c_int, i64, i64, fp, fp] + [fp] * 10 + [fp, ctypes.c_int, ctypes.c_int]
            + [fp] * 6 + [ctypes.c_float, ctypes.c_float, ctypes.c_int, dp, i64,
                          ctypes.c_double, i64, i64, fp, fp]
        )
        L.lo_fused_apply.restype = ctypes.c_int
        L.lo_opt_step.argtypes = [
            ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
            ctypes.c_float, ctypes.c_float, ctypes.c_int, dp, ctypes.c_double,
            ctypes.c_double, fp, i64, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
        ]
        L.lo_opt_step.restype = ctypes.c_int
        L.lo_expf_array.argtypes = [fp, fp, i64]
        L.lo_expf_array.restype = None
        _lib = L
    return _lib


def _f(a):
    assert a.dtype == np.float32 and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _d(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


# ---------------------------------------------------------------------------
# data


@dataclass
class OState:
    """Mirror of state.py:43-74 OptState (f32 arrays, t = step counter)."""

    M: list
    V: np.ndarray
    r: list
    c: list
    t: int = 0

    @classmethod
    def zeros(cls, m, n):
        return cls(
            M=[np.zeros((m, n), F32) for _ in range(3)],
            V=np.zeros((m, n), F32),
            r=[np.zeros(m, F32) for _ in range(3)],
            c=[np.zeros(n, F32) for _ in range(3)],
            t=0,
        )

    def copy(self):
        return OState(M=[a.copy() for a in self.M], V=self.V.copy(),
                      r=[a.copy() for a in self.r], c=[a.copy() for a in self.c], t=self.t)

    @property
    def shape(self):
        return self.V.shape

    def ptrs(self):
        return [_f(a) for a in self.M] + [_f(self.V)] + [_f(a) for a in self.r] + [
            _f(a) for a in self.c]


@dataclass
class Weights:
    """Mirror of engine.py:119-163 LoptWeights for the three-layer MLP."""

    layers: list
    alpha: float = 0.01
    beta_out: float = 0.01
    betas: tuple = DEFAULT_BETAS
    update_sign: int = -1

    def __post_init__(self):
        self.layers = [(np.ascontiguousarray(w, F32), np.ascontiguousarray(b, F32))
                       for w, b in self.layers]

    @property
    def input_dim(self):
        return self.layers[0][0].shape[1]


def random_weights(d_feat, hidden=(32, 32), seed=0, scale=0.2, betas=DEFAULT_BETAS):
    """engine.py:178-192, same generator calls in the same order."""
    rng = np.random.default_rng(seed)
    dims = (d_feat, *hidden, 2)
    layers = []
    for i in range(len(dims) - 1):
        w = rng.standard_normal((dims[i + 1], dims[i]), dtype=F32) * F32(scale)
        b = rng.standard_normal(dims[i + 1], dtype=F32) * F32(scale * 0.5)
        layers.append((w, b))
    return Weights(layers=layers, betas=betas)


def zero_weights(d_feat, hidden=(32, 32)):
    dims = (d_feat, *hidden, 2)
    return Weights(layers=[(np.zeros((dims[i + 1], dims[i]), F32), np.zeros(dims[i + 1], F32))
                           for i in range(len(dims) - 1)])


def time_features(t, kind):
    """features.py:125-130 (numpy tanh, evaluated exactly as the reference)."""
    if kind != SMALL_FC_LOPT:
        return np.zeros(11, F32)
    xs = np.array(TIME_XS, dtype=F32)
    return np.ascontiguousarray(np.tanh(F32(t) / xs).astype(F32))


def schedule_lr(kind, max_lr, min_lr, warmup, total, step):
    """optim.py:69-89."""
    if step < 0:
        raise ValueError("negative step")
    if kind == "constant":
        return max_lr
    if step <= warmup:
        if warmup == 0:
            return max_lr
        return max_lr * (step / warmup)
    if step >= total:
        return min_lr
    progress = (step - warmup) / (total - warmup)
    return min_lr + 0.5 * (max_lr - min_lr) * (1.0 + math.cos(math.pi * progress))


# ---------------------------------------------------------------------------
# per-tensor ops


def state_step(s: OState, g, betas=DEFAULT_BETAS) -> OState:
    g = np.ascontiguousarray(g, F32)
    out = s.copy()
    m, n = out.shape
    st = lib().lo_state_step(m, n, _f(g), *out.ptrs(), _d(np.asarray(betas, np.float64)))
    if st != OK:
        raise OracleError(st)
    out.t = s.t + 1
    return out


def libm_expf(x):
    """glibc expf elementwise (the exp numba uses, engine.py:537)."""
    x = np.ascontiguousarray(x, F32)
    y = np.empty_like(x)
    lib().lo_expf_array(_f(x), _f(y), x.size)
    return y


def factor_means(s: OState):
    m = s.shape[0]
    return tuple(F32(lib().lo_factor_mean(_f(s.r[i]), m)) for i in range(3))


def features_at(idx, W, g, s: OState, kind):
    m, n = s.shape
    d = 39 if kind == SMALL_FC_LOPT else 29
    out = np.zeros(d, F32)
    tf = time_features(s.t, kind)
    lib().lo_features_at(kind, m, n, _f(W), _f(g), *s.ptrs(), _f(tf), idx, _f(out))
    return out


def fused_stats(W, g, s: OState, kind, workers=1, lo=None, hi=None):
    m, n = s.shape
    lo = 0 if lo is None else lo
    hi = m * n if hi is None else hi
    d = 39 if kind == SMALL_FC_LOPT else 29
    sumsq = np.zeros(d, np.float64)
    tf = time_features(s.t, kind)
    st = lib().lo_fused_stats(kind, m, n, _f(W), _f(g), *s.ptrs(), _f(tf), lo, hi, workers,
                              _d(sumsq))
    if st != OK:
        raise OracleError(st)
    return sumsq, hi - lo


def normalization_scale(sumsq, count):
    sumsq = np.ascontiguousarray(sumsq, np.float64)
    out = np.zeros(sumsq.shape[0], F32)
    lib().lo_normalization_scale(sumsq.shape[0], _d(sumsq), count, _f(out))
    return out


def fused_apply(W, g, s: OState, w: Weights, kind, sumsq, count, lr=1.0, lo=None, hi=None,
                out=None):
    m, n = s.shape
    lo = 0 if lo is None else lo
    hi = m * n if hi is None else hi
    out = np.empty((m, n), F32) if out is None else out
    tf = time_features(s.t, kind)
    (w1, b1), (w2, b2), (w3, b3) = w.layers
    maxabs = np.zeros(1, F32)
    st = lib().lo_fused_apply(
        kind, m, n, _f(W), _f(g), *s.ptrs(), _f(tf), w1.shape[0], w2.shape[0],
        _f(w1), _f(b1), _f(w2), _f(b2), _f(w3), _f(b3), F32(w.alpha), F32(w.beta_out),
        int(w.update_sign), _d(np.ascontiguousarray(sumsq, np.float64)), count, float(lr),
        lo, hi, _f(out), _f(maxabs))
    if st != OK:
        raise OracleError(st)
    return out, float(maxabs[0])


def step_fused(W, g, s: OState, w: Weights, kind, lr=1.0, workers=1):
    """engine.py:713-748: state must already be advanced for g."""
    W = np.ascontiguousarray(W, F32)
    g = np.ascontiguousarray(g, F32)
    sumsq, count = fused_stats(W, g, s, kind, workers=workers)
    out, maxabs = fused_apply(W, g, s, w, kind, sumsq, count, lr=lr)
    if not np.isfinite(out).all():
        raise OracleError(ERR_OVERFLOW)
    return out, maxabs, sumsq


# ---------------------------------------------------------------------------
# multi-tensor step


class _Desc(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("n", ctypes.c_int64)] + [
        (name, ctypes.c_void_p) for name in
        ("W", "g", "M0", "M1", "M2", "V", "r0", "r1", "r2", "c0", "c1", "c2",
         "w1", "b1", "w2", "b2", "w3", "b3")]


def opt_step(params, states, grads, weights, kind, lr, weight_decay=0.0, workers=1,
             threads=0, per_tensor_weights=None):
    """optim.py:144-180 over lists of (m, n) f32 arrays, IN PLACE on params and
    states (states' t is bumped).  `lr` is the already-scheduled learning rate
    (schedule_lr at the pre-increment counter).  Tensors run on `threads`
    OpenMP threads (0 = all)."""
    count = len(params)
    descs = (_Desc * max(count, 1))()
    keep = []
    t_new = states[0].t + 1 if states else 1
    tf = time_features(t_new, kind)
    h1 = weights.layers[0][0].shape[0]
    h2 = weights.layers[1][0].shape[0]
    for j in range(count):
        W, g, s = params[j], np.ascontiguousarray(grads[j], F32), states[j]
        assert W.dtype == F32 and W.flags.c_contiguous and W.shape == s.shape
        w = weights if per_tensor_weights is None else per_tensor_weights[j]
        keep.append(g)
        d = descs[j]
        d.m, d.n = s.shape
        d.W, d.g = W.ctypes.data, g.ctypes.data
        d.M0, d.M1, d.M2 = (a.ctypes.data for a in s.M)
        d.V = s.V.ctypes.data
        d.r0, d.r1, d.r2 = (a.ctypes.data for a in s.r)
        d.c0, d.c1, d.c2 = (a.ctypes.data for a in s.c)
        (w1, b1), (w2, b2), (w3, b3) = w.layers
        d.w1, d.b1, d.w2, d.b2, d.w3, d.b3 = (a.ctypes.data for a in (w1, b1, w2, b2, w3, b3))
    err = ctypes.c_int(-1)
    st = lib().lo_opt_step(
        kind, count, ctypes.cast(descs, ctypes.c_void_p), h1, h2, F32(weights.alpha),
        F32(weights.beta_out), int(weights.update_sign),
        _d(np.asarray(weights.betas, np.float64)), float(lr), float(weight_decay), _f(tf),
        workers, threads, ctypes.byref(err))
    if st != OK:
        raise OracleError(st, err.value)
    for s in states:
        s.t += 1


def view_2d(shape):
    """2-D view of a parameter shape.  Rank <= 2 follows tensors.py:66-100
    exactly (0-D -> (1,1), 1-D -> (n,1), 2-D unchanged).  The reference rejects
    rank > 2 (tensors.py:77-78); for those this build drops leading 1s while
    the rank exceeds 2 and then flattens to (d0, prod(rest)) -- the rule
    SURVEY.md section 7.3(6) recommends, applied identically on both sides."""
    shape = tuple(int(s) for s in shape)
    while len(shape) > 2 and shape[0] == 1:
        shape = shape[1:]
    if len(shape) == 0:
        return (1, 1)
    if len(shape) == 1:
        return (shape[0], 1)
    if len(shape) == 2:
        return shape
    rest = 1
    for s in shape[1:]:
        rest *= s
    return (shape[0], rest)


# ---------------------------------------------------------------------------
# The reference's baseline optimizers, restated with
# explicit f32 scalars: every array op below is one correctly rounded f32
# operation, in the reference's order.

def adam_step(theta, g, m, v, beta1=0.9, beta2=0.999, lr=1e-3, eps=1e-8, t=1):
    """pkg/src/lopt/optim.py:187-198.  Returns (theta', m', v')."""
    if t < 1:
        raise ValueError("Adam step count starts at 1")
    one = F32(1.0)
    b1, b2 = F32(beta1), F32(beta2)
    th, gr = np.asarray(theta, F32), np.asarray(g, F32)
    m_new = np.add(np.multiply(b1, m, dtype=F32), np.multiply(one - b1, gr, dtype=F32), dtype=F32)
    g2 = np.multiply(gr, gr, dtype=F32)
    v_new = np.add(np.multiply(b2, v, dtype=F32), np.multiply(one - b2, g2, dtype=F32), dtype=F32)
    c1 = one - b1 ** F32(t)   # numpy's f32 *scalar* power, as the reference (the
    c2 = one - b2 ** F32(t)   # array ufunc path can round differently)
    mh = np.divide(m_new, c1, dtype=F32)
    vh = np.divide(v_new, c2, dtype=F32)
    den = np.add(np.sqrt(vh, dtype=F32), F32(eps), dtype=F32)
    step = np.divide(np.multiply(F32(lr), mh, dtype=F32), den, dtype=F32)
    return np.subtract(th, step, dtype=F32), m_new, v_new


def adafactor_step(theta, g, r, c, beta=0.999, lr=1e-3, eps=1e-30):
    """pkg/src/lopt/optim.py:201-217 with update_adafactor (state.py:93-113)
    and adafactor_scale (features.py:357-362).  Returns (theta', r', c')."""
    gr = np.asarray(g, F32)
    rows, cols = gr.shape
    if rows == 0 or cols == 0:
        raise ValueError("adafactor factors undefined for empty tensors")
    sq = gr.astype(np.float64) ** 2                     # exact: f32 squares fit in f64
    row_mean = (sq.sum(axis=1) / cols).astype(F32)      # numpy mean = sum / count, f64
    col_mean = (sq.sum(axis=0) / rows).astype(F32)
    b = F32(beta)
    omb = F32(1.0) - b
    r_new = np.add(np.multiply(b, r, dtype=F32), np.multiply(omb, row_mean, dtype=F32), dtype=F32)
    c_new = np.add(np.multiply(b, c, dtype=F32), np.multiply(omb, col_mean, dtype=F32), dtype=F32)
    # np.mean(r, dtype=f64) casts in 8192-element buffers; one buffer (this
    # form) for rows <= 8192, which covers the golden cases
    mean_r = F32(r_new.astype(np.float64).sum() / rows)
    outer = np.multiply(r_new[:, None], c_new[None, :], dtype=F32)
    S = np.sqrt(np.divide(mean_r, np.add(outer, F32(eps), dtype=F32), dtype=F32), dtype=F32)
    upd = np.multiply(np.multiply(F32(lr), gr, dtype=F32), S, dtype=F32)
    return np.subtract(np.asarray(theta, F32), upd, dtype=F32), r_new, c_new
