"""Learning-rate schedule and decoupled weight decay (optim.py:52-101)."""

from __future__ import annotations

import math
from dataclasses import dataclass


@dataclass
class ScheduleConfig:
    kind: str = "constant"  # constant | cosine
    max_lr: float = 1.0
    min_lr: float = 0.0
    warmup_steps: int = 0
    total_steps: int = 1

    def __post_init__(self):
        if self.kind not in ("constant", "cosine"):
            raise ValueError(f"unknown schedule kind {self.kind!r}")
        if not 0.0 <= self.min_lr <= self.max_lr:
            raise ValueError(f"need 0 <= min_lr <= max_lr, got {self.min_lr}, {self.max_lr}")
        if not 0 <= self.warmup_steps <= self.total_steps:
            raise ValueError("need 0 <= warmup_steps <= total_steps")


def schedule_lr(cfg: ScheduleConfig, step: int) -> float:
    """optim.py:69-89: constant, or linear warmup then cosine to min_lr,
    with exact endpoints; sampled at the PRE-increment step counter."""
    if step < 0:
        raise ValueError("negative step")
    if cfg.kind == "constant":
        return cfg.max_lr
    if step <= cfg.warmup_steps:
        if cfg.warmup_steps == 0:
            return cfg.max_lr
        return cfg.max_lr * (step / cfg.warmup_steps)
    if step >= cfg.total_steps:
        return cfg.min_lr
    progress = (step - cfg.warmup_steps) / (cfg.total_steps - cfg.warmup_steps)
    return cfg.min_lr + 0.5 * (cfg.max_lr - cfg.min_lr) * (1.0 + math.cos(math.pi * progress))


def decay_factor(lr: float, decay: float):
    """optim.py:92-101: decay is one f32 multiply by f32(1 - lr*decay)."""
    import numpy as np

    if decay < 0:
        raise ValueError("negative weight decay")
    return np.float32(1.0 - lr * decay)
