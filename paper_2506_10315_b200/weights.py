"""Learned-optimizer MLP weights (the reference's LoptWeights).

Mirrors pkg/src/lopt/engine.py:119-228: layers (out, in) with ReLU between
them and (direction, magnitude) out of the last, the update constants alpha,
beta_out and update_sign, and the accumulator betas.  random_weights uses the
same generator calls in the same order as engine.py:178-192, so a seed gives
the reference's exact weights.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

F32 = np.float32


@dataclass(frozen=True)
class BetaConfig:
    """state.py:25-40."""

    momentum_betas: tuple = (0.1, 0.5, 0.9)
    second_moment_beta: float = 0.999
    adafactor_betas: tuple = (0.9, 0.99, 0.999)

    def __post_init__(self):
        for b in (*self.momentum_betas, self.second_moment_beta, *self.adafactor_betas):
            if not 0.0 <= b <= 1.0:
                raise ValueError(f"beta {b} outside [0, 1]")

    def as_tuple(self):
        return (*self.momentum_betas, self.second_moment_beta, *self.adafactor_betas)


@dataclass
class LoptWeights:
    layers: list
    alpha: float = 0.01
    beta_out: float = 0.01
    betas: BetaConfig = field(default_factory=BetaConfig)
    update_sign: int = -1

    def __post_init__(self):
        if not self.layers:
            raise ValueError("empty MLP")
        self.layers = [(np.ascontiguousarray(w, dtype=F32), np.ascontiguousarray(b, dtype=F32))
                       for w, b in self.layers]
        for i, (w, b) in enumerate(self.layers):
            if w.ndim != 2 or b.ndim != 1 or w.shape[0] != b.shape[0]:
                raise ValueError(f"layer {i}: weight {w.shape} / bias {b.shape} mismatch")
            if i > 0 and w.shape[1] != self.layers[i - 1][0].shape[0]:
                raise ValueError(f"layer {i} input dim {w.shape[1]} breaks the chain")
        if self.layers[-1][0].shape[0] != 2:
            raise ValueError("last layer must emit (direction, magnitude)")
        if self.update_sign not in (-1, 1):
            raise ValueError("update_sign must be -1 or +1")

    @property
    def input_dim(self) -> int:
        return self.layers[0][0].shape[1]

    @property
    def n_layers(self) -> int:
        return len(self.layers)

    @property
    def hidden(self) -> tuple:
        return tuple(w.shape[0] for w, _ in self.layers[:-1])

    def packed(self) -> np.ndarray:
        """w1 | b1 | w2 | b2 | w3 | b3, the layout of lopt_set_weights."""
        if self.n_layers != 3:
            # engine.py:676-680: the streaming path supports exactly 3 layers
            raise ValueError(f"the fused path supports the three-layer MLP; got {self.n_layers}")
        return np.concatenate([a.ravel() for wb in self.layers for a in wb]).astype(F32)


def zero_weights(d_feat, hidden=(32, 32), betas=None) -> LoptWeights:
    dims = (d_feat, *hidden, 2)
    layers = [(np.zeros((dims[i + 1], dims[i]), F32), np.zeros(dims[i + 1], F32))
              for i in range(len(dims) - 1)]
    return LoptWeights(layers=layers, betas=betas or BetaConfig())


def random_weights(d_feat, hidden=(32, 32), seed=0, scale=0.2, betas=None) -> LoptWeights:
    rng = np.random.default_rng(seed)
    dims = (d_feat, *hidden, 2)
    layers = []
    for i in range(len(dims) - 1):
        w = rng.standard_normal((dims[i + 1], dims[i]), dtype=F32) * F32(scale)
        b = rng.standard_normal(dims[i + 1], dtype=F32) * F32(scale * 0.5)
        layers.append((w, b))
    return LoptWeights(layers=layers, betas=betas or BetaConfig())


def unpack(packed: np.ndarray, d_feat: int, hidden=(32, 32), **kw) -> LoptWeights:
    h1, h2 = hidden
    sizes = [(h1, d_feat), (h1,), (h2, h1), (h2,), (2, h2), (2,)]
    arrs, off = [], 0
    for s in sizes:
        n = int(np.prod(s))
        arrs.append(np.asarray(packed[off:off + n], F32).reshape(s))
        off += n
    return LoptWeights(layers=[(arrs[0], arrs[1]), (arrs[2], arrs[3]), (arrs[4], arrs[5])], **kw)
