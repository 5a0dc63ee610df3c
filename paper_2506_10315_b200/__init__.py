"""B200-native learned-optimizer step (PyLO small_fc_lopt / VeLO) behind the
torch.optim surface, with sm_100a kernels reached through a C ABI
(include/lopt_b200.h).  See DESIGN.md."""

from .engine import (DeviceOptState, EngineError, FeatureStats, Slot, StepPlan, UpdateOverflowError,
                     fast_available, fused_apply, fused_stats, step_fused, step_naive,
                     UpdateReport)
from .features import (FeatureSet, FeatureSetSpec, column_names, small_fc_lopt_spec,
                       spec_by_name, time_features, velo_mlp_spec)
from .optim import AdafacLO_CUDA, LearnedOptimizer, OptimError, opt_step, view_2d
from .schedule import ScheduleConfig, schedule_lr
from .velo import VeLO_CUDA, VeLOHyperNet
from .weights import BetaConfig, LoptWeights, random_weights, zero_weights

__all__ = [
    "AdafacLO_CUDA", "BetaConfig", "column_names", "DeviceOptState", "EngineError",
    "fast_available", "FeatureSet", "FeatureSetSpec", "FeatureStats", "fused_apply",
    "fused_stats", "LearnedOptimizer", "LoptWeights", "opt_step", "OptimError", "random_weights",
    "schedule_lr", "ScheduleConfig", "Slot", "small_fc_lopt_spec", "spec_by_name",
    "step_fused", "step_naive", "StepPlan", "time_features", "UpdateOverflowError", "UpdateReport",
    "VeLO_CUDA", "velo_mlp_spec", "VeLOHyperNet", "view_2d", "zero_weights",
]
