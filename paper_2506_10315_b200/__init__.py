"""B200-native learned-optimizer step (PyLO small_fc_lopt / VeLO) behind the
torch.optim surface, with sm_100a kernels reached through a C ABI
(include/lopt_b200.h).  See DESIGN.md."""

from .engine import (DeviceOptState, EngineError, FeatureStats, Slot, StepPlan, UpdateOverflowError,
                     fast_available, fused_apply, fused_stats, step_fused, step_naive)
from .features import (FeatureSet, FeatureSetSpec, column_names, small_fc_lopt_spec,
                       spec_by_name, time_features, velo_mlp_spec)
from .optim import AdafacLO_CUDA, LearnedOptimizer, OptimError, view_2d
from .schedule import ScheduleConfig, schedule_lr
from .velo import VeLO_CUDA, VeLOHyperNet
from .weights import BetaConfig, LoptWeights, random_weights, zero_weights

__all__ = [
    "AdafacLO_CUDA", "BetaConfig", "DeviceOptState", "EngineError", "FeatureSet",
    "FeatureSetSpec", "LearnedOptimizer", "LoptWeights", "OptimError", "ScheduleConfig", "Slot",
    "StepPlan", "UpdateOverflowError", "column_names", "FeatureStats", "fused_apply", "fused_stats", "random_weights",
    "schedule_lr", "small_fc_lopt_spec", "spec_by_name", "step_fused", "step_naive", "time_features",
    "velo_mlp_spec", "view_2d", "zero_weights",
]
