"""Feature-set specs and the per-step host scalars.

Mirrors pkg/src/lopt/features.py:52-140 of the reference: the frozen column
orders of small_fc_lopt (39) and VELO_MLP (29), the eps constants, and the
host-side time features.  The per-element feature arithmetic itself lives in
the CUDA kernels (csrc/lopt_common.cuh strict_features, csrc/lopt_fast.cu).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _lib

F32 = np.float32

TIME_XS = (1.0, 3.0, 10.0, 30.0, 100.0, 300.0, 1000.0, 3000.0, 1e4, 3e4, 1e5)


class FeatureSet(enum.Enum):
    SMALL_FC_LOPT = "small_fc_lopt"
    VELO_MLP = "velo_mlp"


@dataclass(frozen=True)
class FeatureSetSpec:
    """features.py:60-72."""

    id: FeatureSet
    d_feat: int
    time_xs: tuple
    clip_bound: float | None
    eps_recip: float = 1e-12
    eps_norm: float = 1e-5

    def __post_init__(self):
        expected = 39 if self.id is FeatureSet.SMALL_FC_LOPT else 29
        if self.d_feat != expected:
            raise ValueError(f"{self.id.value} must have {expected} columns, got {self.d_feat}")

    @property
    def abi_kind(self) -> int:
        return _lib.LOPT_SMALL_FC_LOPT if self.id is FeatureSet.SMALL_FC_LOPT else _lib.LOPT_VELO_MLP


def small_fc_lopt_spec() -> FeatureSetSpec:
    return FeatureSetSpec(id=FeatureSet.SMALL_FC_LOPT, d_feat=39, time_xs=TIME_XS, clip_bound=None)


def velo_mlp_spec() -> FeatureSetSpec:
    return FeatureSetSpec(id=FeatureSet.VELO_MLP, d_feat=29, time_xs=(), clip_bound=0.1)


def spec_by_name(name: str) -> FeatureSetSpec:
    for fs, factory in ((FeatureSet.SMALL_FC_LOPT, small_fc_lopt_spec),
                        (FeatureSet.VELO_MLP, velo_mlp_spec)):
        if name == fs.value:
            return factory()
    raise ValueError(f"unknown feature set {name!r}")


def column_names(spec: FeatureSetSpec) -> list[str]:
    base = (
        ["M1", "M2", "M3", "V", "r5", "r6", "r7", "c5", "c6", "c7"]
        + ["M1_rsqrtV", "M2_rsqrtV", "M3_rsqrtV", "rsqrt_V"]
        + ["rsqrt_r5", "rsqrt_r6", "rsqrt_r7", "rsqrt_c5", "rsqrt_c6", "rsqrt_c7"]
        + ["g_adafac5", "g_adafac6", "g_adafac7", "M1_adafac5", "M2_adafac6", "M3_adafac7"]
    )
    if spec.id is FeatureSet.SMALL_FC_LOPT:
        return base + [f"tanh_t_{x:g}" for x in spec.time_xs] + ["W", "g"]
    return base + ["W", "g", "g_clipped"]


def time_features(t: int, spec: FeatureSetSpec) -> np.ndarray:
    """features.py:125-130: tanh(f32(t)/x) in f32, evaluated with numpy on the
    host exactly as the reference does (numpy's f32 tanh is not CUDA tanhf).
    Always returns 11 values (zeros for feature sets without time columns)."""
    if not spec.time_xs:
        return np.zeros(11, dtype=F32)
    xs = np.array(spec.time_xs, dtype=F32)
    return np.tanh(F32(t) / xs).astype(F32)
