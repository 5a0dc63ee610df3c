"""ctypes binding of the sm_100a C-ABI library (include/lopt_b200.h).

There is no CPU fallback: if the library is missing, cannot be loaded, or no
CUDA device is present, every entry point raises LoptUnavailableError.
"""

from __future__ import annotations

import ctypes
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# LOPT_SO: an alternative build of the same library (tuning experiments only)
SO = os.environ.get("LOPT_SO") or os.path.join(PKG, "_lib", "liblopt_b200.so")

LOPT_OK = 0
LOPT_ERR_INVALID = 1
LOPT_ERR_SHAPE = 2
LOPT_ERR_WORKSPACE = 3
LOPT_ERR_CUDA = 4
LOPT_ERR_UNSUPPORTED = 5

LOPT_SMALL_FC_LOPT = 0
LOPT_VELO_MLP = 1
LOPT_MODE_STRICT = 0
LOPT_MODE_FAST = 1
LOPT_STATUS_NONFINITE_GRAD = 1
LOPT_STATUS_NONFINITE_PARAM = 2

EXPORTS = [
    "lopt_plan_create", "lopt_plan_destroy", "lopt_workspace_bytes", "lopt_bind_workspace",
    "lopt_rebind_tensors", "lopt_set_weights", "lopt_weights_ptr", "lopt_set_step_args",
    "lopt_factor_partials", "lopt_factor_finalize", "lopt_feature_stats", "lopt_apply",
    "lopt_step", "lopt_factor_sums_ptr", "lopt_stat_sums_ptr", "lopt_status_ptr",
    "lopt_read_status", "lopt_debug_ptrs", "lopt_version",
    "lopt_num_kernels_launched_last_step", "lopt_velo_mix", "lopt_selftest_umma",
    "lopt_probe_umma", "lopt_selftest_expf", "lopt_set_peers", "lopt_graph_step",
    "lopt_graph_reset", "lopt_set_velo", "lopt_probe_tmem", "lopt_adam_step",
    "lopt_adafactor_step", "lopt_adafactor_scratch_bytes", "lopt_set_stat_counts",
    "lopt_enable_peer_access", "lopt_set_phase_timing", "lopt_phase_slot",
    "lopt_phase_elapsed",
]


class LoptError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        names = {1: "invalid argument", 2: "shape error", 3: "workspace too small",
                 4: "CUDA error", 5: "unsupported configuration"}
        super().__init__(f"lopt_b200 {what}: {names.get(code, code)}")


class LoptUnavailableError(RuntimeError):
    """The CUDA extension is missing or unusable; there is no fallback."""


class lopt_tensor(ctypes.Structure):
    _fields_ = [
        ("m", ctypes.c_int64), ("n", ctypes.c_int64), ("lo", ctypes.c_int64),
        ("hi", ctypes.c_int64), ("theta", ctypes.c_void_p), ("grad", ctypes.c_void_p),
        ("state", ctypes.c_void_p), ("row_factors", ctypes.c_void_p),
        ("col_factors", ctypes.c_void_p), ("weight_slot", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class lopt_config(ctypes.Structure):
    _fields_ = [
        ("feature_set", ctypes.c_int32), ("mode", ctypes.c_int32),
        ("hidden1", ctypes.c_int32), ("hidden2", ctypes.c_int32),
        ("num_weight_sets", ctypes.c_int32), ("state_advanced", ctypes.c_int32),
        ("betas", ctypes.c_double * 7), ("alpha", ctypes.c_float), ("beta_out", ctypes.c_float),
        ("update_sign", ctypes.c_int32), ("reserved", ctypes.c_int32),
    ]


class lopt_step_args(ctypes.Structure):
    _fields_ = [
        ("lr", ctypes.c_double), ("weight_decay", ctypes.c_double),
        ("time_features", ctypes.c_float * 11), ("t", ctypes.c_int32),
        ("loss_features", ctypes.c_float * 2),
    ]


_lib = None


def lib(required: bool = True):
    """Load the shared library (building it first in a source checkout)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(SO) or os.environ.get("LOPT_REBUILD"):
        try:
            from . import build as _build

            _build.build()
        except Exception as e:  # noqa: BLE001
            if required:
                raise LoptUnavailableError(f"cannot build {SO}: {e}") from e
            return None
    try:
        L = ctypes.CDLL(SO)
    except OSError as e:
        if required:
            raise LoptUnavailableError(f"cannot load {SO}: {e}") from e
        return None
    vp = ctypes.c_void_p
    i32 = ctypes.c_int32
    L.lopt_plan_create.argtypes = [ctypes.POINTER(lopt_tensor), i32, ctypes.POINTER(lopt_config),
                                   ctypes.POINTER(vp)]
    L.lopt_plan_destroy.argtypes = [vp]
    L.lopt_workspace_bytes.argtypes = [vp, ctypes.POINTER(ctypes.c_size_t)]
    L.lopt_bind_workspace.argtypes = [vp, vp, ctypes.c_size_t, vp]
    L.lopt_rebind_tensors.argtypes = [vp, ctypes.POINTER(lopt_tensor), i32, vp]
    L.lopt_set_weights.argtypes = [vp, i32, vp, i32, vp]
    L.lopt_weights_ptr.argtypes = [vp, i32, ctypes.POINTER(vp)]
    L.lopt_set_step_args.argtypes = [vp, ctypes.POINTER(lopt_step_args), vp]
    for name in ("lopt_factor_partials", "lopt_factor_finalize", "lopt_feature_stats",
                 "lopt_apply"):
        getattr(L, name).argtypes = [vp, vp]
    L.lopt_step.argtypes = [vp, ctypes.POINTER(lopt_step_args), vp]
    L.lopt_factor_sums_ptr.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_int64)]
    L.lopt_stat_sums_ptr.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(ctypes.c_int64)]
    L.lopt_status_ptr.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]
    L.lopt_read_status.argtypes = [vp, vp, vp, vp]
    L.lopt_debug_ptrs.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]
    L.lopt_version.restype = ctypes.c_char_p
    L.lopt_num_kernels_launched_last_step.argtypes = [vp]
    L.lopt_velo_mix.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp, vp]
    L.lopt_selftest_umma.argtypes = [i32, i32, vp, vp, vp, vp]
    L.lopt_probe_umma.argtypes = [i32, i32, vp, vp]
    L.lopt_probe_tmem.argtypes = [i32, i32, i32, i32, vp, vp]
    L.lopt_adam_step.argtypes = [vp, vp, vp, vp, ctypes.c_int64, vp, vp]
    L.lopt_adafactor_step.argtypes = [vp, vp, vp, vp, ctypes.c_int64, ctypes.c_int64, vp, vp, vp]
    L.lopt_adafactor_scratch_bytes.argtypes = [ctypes.c_int64, ctypes.c_int64]
    L.lopt_set_stat_counts.argtypes = [vp, vp, vp]
    L.lopt_enable_peer_access.argtypes = [i32]
    L.lopt_set_peers.argtypes = [vp, i32, vp]
    L.lopt_selftest_expf.argtypes = [vp, vp, ctypes.c_int64, vp]
    L.lopt_graph_step.argtypes = [vp, ctypes.POINTER(lopt_step_args), vp]
    L.lopt_graph_reset.argtypes = [vp]
    L.lopt_set_phase_timing.argtypes = [vp, i32]
    L.lopt_phase_slot.argtypes = [vp, ctypes.POINTER(i32)]
    L.lopt_phase_elapsed.argtypes = [vp, i32, i32, i32, ctypes.POINTER(ctypes.c_float)]
    L.lopt_set_velo.argtypes = [vp, vp, vp, vp, vp, i32, i32, vp]
    for name in EXPORTS:
        f = getattr(L, name)
        if name != "lopt_version":
            f.restype = ctypes.c_int
    L.lopt_adafactor_scratch_bytes.restype = ctypes.c_int64
    _lib = L
    return L


def check(code: int, what: str = ""):
    if code != LOPT_OK:
        raise LoptError(code, what)


def require_cuda():
    import torch

    if not torch.cuda.is_available():
        raise LoptUnavailableError("the B200 learned-optimizer step needs a CUDA device; "
                                   "there is no CPU fallback")
    return lib()
