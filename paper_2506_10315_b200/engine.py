"""Device engine: a step plan over a list of CUDA tensors, and the reference's
engine-level functions on top of it.

StepPlan wraps one lopt_plan (include/lopt_b200.h): the tensors' 2-D views and
element ranges, a workspace carved out of the torch caching allocator, and the
MLP weight slots.  The functional API mirrors pkg/src/lopt/engine.py:

    fused_stats(W, g, state, spec)              engine.py:619-654
    fused_apply(W, g, state, weights, spec, stats, out, lr)   engine.py:657-710
    step_fused(W, g, state, weights, spec, lr)  engine.py:713-748

where `state` is already advanced for g (the reference's precondition), and
`opt_step`-level work (state advance fused into the passes, schedules, decay)
lives in optim.py.
"""

from __future__ import annotations

import ctypes
from typing import NamedTuple
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .features import FeatureSetSpec, small_fc_lopt_spec, time_features
from .weights import BetaConfig, LoptWeights

F32 = np.float32


class EngineError(Exception):
    """engine.py:65-66."""


class UpdateOverflowError(EngineError):
    """engine.py:84-85: the update produced non-finite values."""


def _stream_handle(stream=None) -> int:
    if stream is not None:
        return stream.cuda_stream
    return torch.cuda.current_stream().cuda_stream


@dataclass
class Slot:
    """One tensor as the kernels see it.  theta/grad: contiguous f32 CUDA
    tensors of m*n elements; state: (hi-lo, 4) f32 {M1, M2, M3, V}; r: (3, m),
    c: (3, n) f32."""

    theta: torch.Tensor
    grad: torch.Tensor
    state: torch.Tensor
    r: torch.Tensor
    c: torch.Tensor
    m: int
    n: int
    lo: int = 0
    hi: int = -1
    weight_slot: int = 0

    def __post_init__(self):
        if self.hi < 0:
            self.hi = self.m * self.n

    def abi(self) -> _lib.lopt_tensor:
        for name in ("theta", "grad", "state", "r", "c"):
            t = getattr(self, name)
            if t.dtype != torch.float32 or not t.is_cuda or not t.is_contiguous():
                raise TypeError(f"{name} must be a contiguous float32 CUDA tensor")
        if self.theta.numel() != self.m * self.n or self.grad.numel() != self.m * self.n:
            raise EngineError(f"shape mismatch: param/grad vs ({self.m}, {self.n})")
        if self.state.numel() < 4 * (self.hi - self.lo):
            raise EngineError("state buffer smaller than the stepped range")
        return _lib.lopt_tensor(
            m=self.m, n=self.n, lo=self.lo, hi=self.hi, theta=self.theta.data_ptr(),
            grad=self.grad.data_ptr(), state=self.state.data_ptr(), row_factors=self.r.data_ptr(),
            col_factors=self.c.data_ptr(), weight_slot=self.weight_slot, reserved=0)


class PhaseMark:
    """One of a timed step's phase events (StepPlan.step_timed); like
    torch.cuda.Event.elapsed_time, in ms."""

    def __init__(self, plan, slot: int, k: int):
        self.plan, self.slot, self.k = plan, slot, k

    def elapsed_time(self, other: "PhaseMark") -> float:
        ms = ctypes.c_float()
        _lib.check(self.plan.L.lopt_phase_elapsed(self.plan.h, self.slot, self.k, other.k,
                                                  ctypes.byref(ms)), "phase_elapsed")
        return float(ms.value)


class StepPlan:
    """A compiled step over fixed tensors (OptimizerHandle of optim.py:104-141)."""

    def __init__(self, slots, spec: FeatureSetSpec, weights, *, mode="strict",
                 state_advanced=False, device=None):
        self.L = _lib.require_cuda()
        self.spec = spec
        self.slots = list(slots)
        weights_list = weights if isinstance(weights, (list, tuple)) else [weights]
        w0 = weights_list[0]
        if w0.input_dim != spec.d_feat:
            raise EngineError(f"MLP input dim {w0.input_dim} does not match feature set "
                              f"({spec.d_feat} columns)")
        if w0.n_layers != 3:
            raise EngineError("the streaming path supports the reference three-layer MLP "
                              f"topology; got {w0.n_layers} layers")
        self.hidden = w0.hidden
        self.weights = weights_list
        self.mode = mode
        self.device = device or self.slots[0].theta.device
        cfg = _lib.lopt_config()
        cfg.feature_set = spec.abi_kind
        cfg.mode = _lib.LOPT_MODE_FAST if mode == "fast" else _lib.LOPT_MODE_STRICT
        cfg.hidden1, cfg.hidden2 = self.hidden
        cfg.num_weight_sets = len(weights_list)
        cfg.state_advanced = 1 if state_advanced else 0
        for k, b in enumerate(w0.betas.as_tuple()):
            cfg.betas[k] = float(b)
        cfg.alpha = float(F32(w0.alpha))
        cfg.beta_out = float(F32(w0.beta_out))
        cfg.update_sign = int(w0.update_sign)
        self.cfg = cfg
        self._tensors = (_lib.lopt_tensor * len(self.slots))(*[s.abi() for s in self.slots])
        h = ctypes.c_void_p()
        _lib.check(self.L.lopt_plan_create(self._tensors, len(self.slots), ctypes.byref(cfg),
                                           ctypes.byref(h)), "plan_create")
        self.h = h
        nbytes = ctypes.c_size_t()
        _lib.check(self.L.lopt_workspace_bytes(h, ctypes.byref(nbytes)))
        self.ws_bytes = nbytes.value
        self.ws = torch.empty(self.ws_bytes + 256, dtype=torch.uint8, device=self.device)
        base = self.ws.data_ptr()
        self._ws_off = (-base) % 256
        stream = _stream_handle()
        _lib.check(self.L.lopt_bind_workspace(h, base + self._ws_off, self.ws_bytes, stream),
                   "bind_workspace")
        self._packed = []
        for slot, w in enumerate(weights_list):
            self.set_weights(slot, w)
        self._step_args = _lib.lopt_step_args()
        self.graph_steps = 0
        self._tf_t = None
        self._velo_key = None
        # object with .loss_features (the owning optimizer), or None
        self.loss_src = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                torch.cuda.current_stream().synchronize()
            except Exception:  # noqa: BLE001
                pass
            self.L.lopt_plan_destroy(h)
            self.h = None

    # -- configuration ---------------------------------------------------
    def set_weights(self, slot: int, w: LoptWeights):
        packed = torch.from_numpy(w.packed()).to(self.device)
        self._packed.append(packed)  # keep alive until the stream copy ran
        _lib.check(self.L.lopt_set_weights(self.h, slot, packed.data_ptr(), 1, _stream_handle()),
                   "set_weights")

    def weights_ptr(self, slot: int) -> int:
        p = ctypes.c_void_p()
        _lib.check(self.L.lopt_weights_ptr(self.h, slot, ctypes.byref(p)))
        return p.value

    def rebind(self, slots):
        self.slots = list(slots)
        self._tensors = (_lib.lopt_tensor * len(self.slots))(*[s.abi() for s in self.slots])
        _lib.check(self.L.lopt_rebind_tensors(self.h, self._tensors, len(self.slots),
                                              _stream_handle()), "rebind_tensors")

    def set_step(self, lr: float, weight_decay: float, t: int):
        _lib.check(self.L.lopt_set_step_args(self.h, ctypes.byref(self._args(lr, weight_decay, t)),
                                             _stream_handle()), "set_step_args")

    # -- phases ----------------------------------------------------------
    def factor_partials(self):
        _lib.check(self.L.lopt_factor_partials(self.h, _stream_handle()), "factor_partials")

    def factor_finalize(self):
        _lib.check(self.L.lopt_factor_finalize(self.h, _stream_handle()), "factor_finalize")

    def feature_stats(self):
        _lib.check(self.L.lopt_feature_stats(self.h, _stream_handle()), "feature_stats")

    def apply(self):
        _lib.check(self.L.lopt_apply(self.h, _stream_handle()), "apply")

    def _args(self, lr: float, weight_decay: float, t: int):
        args = self._step_args
        args.lr = float(lr)
        args.weight_decay = float(weight_decay)
        # tanh(t/x) for all 11 horizons: the small_fc_lopt columns
        # (features.py:125-130) and the VeLO hypernetwork inputs; the
        # VELO_MLP per-element kernels ignore them
        if t != self._tf_t:
            tf = time_features(t, small_fc_lopt_spec())
            for k in range(11):
                args.time_features[k] = float(tf[k])
            self._tf_t = t
        args.t = int(t)
        # VeLO's loss features travel with the step scalars (no upload)
        src = self.loss_src
        lf = src.loss_features if src is not None else (0.0, 0.0)
        args.loss_features[0] = lf[0]
        args.loss_features[1] = lf[1]
        return args

    def step(self, lr: float, weight_decay: float, t: int):
        _lib.check(self.L.lopt_step(self.h, ctypes.byref(self._args(lr, weight_decay, t)),
                                    _stream_handle()), "step")

    def step_timed(self, lr: float, weight_decay: float, t: int, graph: bool = True,
                   slots: int = 512):
        """step() (graph=False) or graph_step() recording the plan's phase
        events (lopt_set_phase_timing): returns five PhaseMarks -- before the
        factors, after the factors, after the feature statistics, after the
        VeLO hypernetwork, after the apply pass -- whose elapsed_time() is
        valid once the step completed.  A plan keeps `slots` event sets; read
        the marks before that many further timed steps reuse them."""
        if getattr(self, "_ev_slots", 0) == 0:
            _lib.check(self.L.lopt_set_phase_timing(self.h, int(slots)), "set_phase_timing")
            self._ev_slots = int(slots)
        slot = ctypes.c_int32()
        _lib.check(self.L.lopt_phase_slot(self.h, ctypes.byref(slot)), "phase_slot")
        if graph:
            self.graph_step(lr, weight_decay, t)
        else:
            self.step(lr, weight_decay, t)
        return [PhaseMark(self, slot.value, k) for k in range(5)]

    def clear_phase_events(self):
        """Turn phase timing off (the next graph step recaptures without
        event nodes)."""
        if getattr(self, "_ev_slots", 0):
            _lib.check(self.L.lopt_set_phase_timing(self.h, 0), "set_phase_timing")
            self._ev_slots = 0

    def graph_step(self, lr: float, weight_decay: float, t: int):
        """step() replayed from the plan's captured CUDA graph (one launch)."""
        _lib.check(self.L.lopt_graph_step(self.h, ctypes.byref(self._args(lr, weight_decay, t)),
                                          _stream_handle()), "graph_step")
        self.graph_steps += 1

    def gexec_ready(self) -> bool:
        """True once a step ran from the captured graph."""
        return self.graph_steps > 0

    def set_velo(self, hyper, lstm, bank, loss, hidden, bank_size, mix=None):
        """Register the VeLO hypernetwork (device tensors) so step() and
        graph_step() run it between phases 1 and 2; hyper=None unregisters."""
        if hyper is None:
            _lib.check(self.L.lopt_set_velo(self.h, None, None, None, None, 0, 0, None))
            self._velo_key = None
            return
        lp = loss.data_ptr() if loss is not None else None   # None: from the step scalars
        _lib.check(self.L.lopt_set_velo(self.h, hyper.data_ptr(), lstm.data_ptr(),
                                        bank.data_ptr(), lp, int(hidden),
                                        int(bank_size), mix.data_ptr() if mix is not None else None),
                   "set_velo")
        self._velo_key = (hyper.data_ptr(), lstm.data_ptr(), bank.data_ptr(), lp,
                          mix.data_ptr() if mix is not None else None)

    def set_stat_counts(self, counts):
        """Element counts behind each tensor's feature statistics for the
        apply pass's normalization (None: the whole tensors)."""
        if counts is None:
            _lib.check(self.L.lopt_set_stat_counts(self.h, None, _stream_handle()), "set_stat_counts")
            return
        arr = np.asarray(counts, dtype=np.int64)
        _lib.check(self.L.lopt_set_stat_counts(self.h, arr.ctypes.data, _stream_handle()),
                   "set_stat_counts")
        torch.cuda.current_stream().synchronize()   # the host array is a temporary

    def set_peers(self, deltas):
        """Fused parameter all-gather: the apply pass also stores every updated
        parameter at these byte offsets from its local address (the peers'
        mapped parameter arenas).  An empty list disables it."""
        arr = (ctypes.c_int64 * max(1, len(deltas)))(*[int(d) for d in deltas])
        _lib.check(self.L.lopt_set_peers(self.h, len(deltas), arr), "set_peers")

    def local_elements(self) -> int:
        return sum(s.hi - s.lo for s in self.slots)

    def launches_last_step(self) -> int:
        return int(self.L.lopt_num_kernels_launched_last_step(self.h))

    # -- views into the workspace ----------------------------------------
    def _view(self, ptr: int, count: int, dtype) -> torch.Tensor:
        off = ptr - self.ws.data_ptr()
        esize = torch.empty((), dtype=dtype).element_size()
        return self.ws[off:off + count * esize].view(dtype)

    def factor_sums(self) -> torch.Tensor:
        p, c = ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(self.L.lopt_factor_sums_ptr(self.h, ctypes.byref(p), ctypes.byref(c)))
        return self._view(p.value, c.value, torch.float64)

    def stat_sums(self) -> torch.Tensor:
        p, c = ctypes.c_void_p(), ctypes.c_int64()
        _lib.check(self.L.lopt_stat_sums_ptr(self.h, ctypes.byref(p), ctypes.byref(c)))
        return self._view(p.value, c.value, torch.float64).view(len(self.slots), self.spec.d_feat)

    def factor_means(self) -> torch.Tensor:
        p = ctypes.c_void_p()
        _lib.check(self.L.lopt_debug_ptrs(self.h, None, ctypes.byref(p)))
        return self._view(p.value, 4 * len(self.slots), torch.float32).view(-1, 4)[:, :3]

    def status(self, sync=True):
        st = np.zeros(len(self.slots), np.uint32)
        mx = np.zeros(len(self.slots), F32)
        _lib.check(self.L.lopt_read_status(self.h, st.ctypes.data, mx.ctypes.data,
                                           _stream_handle()), "read_status")
        return st, mx


def fast_available() -> bool:
    """True if the library was built with the fast (tensor-core) mode."""
    L = _lib.lib(required=False)
    if L is None:
        return False
    t = _lib.lopt_tensor(m=256, n=256, lo=0, hi=65536, theta=256, grad=256, state=256,
                         row_factors=256, col_factors=256, weight_slot=0, reserved=0)
    cfg = _lib.lopt_config()
    cfg.feature_set = _lib.LOPT_SMALL_FC_LOPT
    cfg.mode = _lib.LOPT_MODE_FAST
    cfg.hidden1 = cfg.hidden2 = 32
    cfg.num_weight_sets = 1
    for k, b in enumerate(BetaConfig().as_tuple()):
        cfg.betas[k] = b
    cfg.update_sign = -1
    h = ctypes.c_void_p()
    rc = L.lopt_plan_create(ctypes.byref(t), 1, ctypes.byref(cfg), ctypes.byref(h))
    if rc == 0:
        L.lopt_plan_destroy(h)
    return rc == 0


# ---------------------------------------------------------------------------
# reference-shaped engine functions (state already advanced)


@dataclass
class DeviceOptState:
    """A device mirror of state.py:43-74 OptState: quad = (m*n, 4)
    {M1, M2, M3, V}, r (3, m), c (3, n), t."""

    quad: torch.Tensor
    r: torch.Tensor
    c: torch.Tensor
    t: int = 0
    shape: tuple = field(default=(0, 0))

    @classmethod
    def zeros(cls, m, n, device="cuda"):
        return cls(quad=torch.zeros(m * n, 4, device=device), r=torch.zeros(3, m, device=device),
                   c=torch.zeros(3, n, device=device), t=0, shape=(m, n))

    @classmethod
    def from_arrays(cls, M, V, r, c, t, device="cuda"):
        m, n = V.shape
        quad = np.stack([np.asarray(M[0]), np.asarray(M[1]), np.asarray(M[2]), np.asarray(V)],
                        axis=-1).reshape(m * n, 4).astype(F32)
        return cls(quad=torch.from_numpy(quad).to(device),
                   r=torch.from_numpy(np.stack([np.asarray(x, F32) for x in r])).to(device),
                   c=torch.from_numpy(np.stack([np.asarray(x, F32) for x in c])).to(device),
                   t=int(t), shape=(m, n))

    def arrays(self):
        m, n = self.shape
        q = self.quad.cpu().numpy().reshape(m, n, 4)
        return ([q[..., 0].copy(), q[..., 1].copy(), q[..., 2].copy()], q[..., 3].copy(),
                [x.copy() for x in self.r.cpu().numpy()], [x.copy() for x in self.c.cpu().numpy()])


def _check_step_inputs(W, g, state, weights, spec):
    """engine.py:583-594."""
    if tuple(W.shape) != tuple(g.shape) or tuple(W.shape) != tuple(state.shape):
        raise EngineError(f"shape mismatch: W {tuple(W.shape)}, g {tuple(g.shape)}, "
                          f"state {tuple(state.shape)}")
    if weights.input_dim != spec.d_feat:
        raise EngineError(f"MLP input dim {weights.input_dim} does not match feature set "
                          f"({spec.d_feat} columns)")
    if W.numel() == 0:
        raise EngineError("empty tensor")


def _engine_plan(W, g, state, weights, spec, mode, lo=None, hi=None):
    m, n = state.shape
    lo = 0 if lo is None else int(lo)
    hi = m * n if hi is None else int(hi)
    if not 0 <= lo <= hi <= m * n:
        raise EngineError(f"element range [{lo}, {hi}) outside a {m}x{n} tensor")
    slot = Slot(theta=W.reshape(-1), grad=g.reshape(-1).contiguous(), state=state.quad[lo:hi],
                r=state.r, c=state.c, m=m, n=n, lo=lo, hi=hi)
    return StepPlan([slot], spec, weights, mode=mode, state_advanced=True)


class FeatureStats(NamedTuple):
    """features.py:107-118: column sums of squared features (f64, here a CUDA
    tensor) and the element count behind them.  Unpacks as (sumsq, count)."""

    sumsq: torch.Tensor
    count: int


def fused_stats(W, g, state: DeviceOptState, spec=None, workers: int = 1, tracker=None,
                lo: int | None = None, hi: int | None = None, mode="strict") -> FeatureStats:
    """engine.py:619-654 pass 1 over the element range [lo, hi) (default: the
    whole tensor).  `workers` and `tracker` are accepted for signature parity:
    `workers` only partitions the reference's f64 reduction and the device
    reduction order is fixed by the plan; device scratch is the plan's own
    workspace (lopt_workspace_bytes), not a tracked host allocation.  Range
    stats add: the sharded step all-reduces them (distsim.py:489-490)."""
    spec = spec or small_fc_lopt_spec()
    from .weights import zero_weights

    plan = _engine_plan(W.detach().clone(), g.detach(), state, zero_weights(spec.d_feat), spec,
                        mode, lo, hi)
    plan.set_step(1.0, 0.0, state.t)
    plan.factor_partials()
    plan.factor_finalize()
    plan.feature_stats()
    count = plan.slots[0].hi - plan.slots[0].lo
    return FeatureStats(plan.stat_sums()[0].clone(), count)


def fused_apply(W, g, state: DeviceOptState, weights: LoptWeights, spec, stats, out,
                lr: float = 1.0, tracker=None, lo: int | None = None, hi: int | None = None,
                mode="strict") -> float:
    """engine.py:657-710 pass 2 over [lo, hi): features normalized by the
    given whole-tensor `stats` (FeatureStats or a (sumsq, count) pair; the
    scale uses the tensor's element count, as the fold at engine.py:686
    does), MLP, update written into out[lo:hi] (a CUDA tensor shaped like W;
    the rest of `out` is not touched).  Returns max |update| over the range.
    The state must already be advanced for g."""
    spec = spec or small_fc_lopt_spec()
    _check_step_inputs(W, g, state, weights, spec)
    if tuple(out.shape) != tuple(W.shape) or not out.is_contiguous():
        raise EngineError(f"out must be a contiguous tensor shaped {tuple(W.shape)}")
    sumsq, count = (stats[0], stats[1]) if isinstance(stats, tuple) else (stats.sumsq, stats.count)
    m, n = state.shape
    if int(count) < 1:
        raise EngineError(f"stats over {int(count)} elements")
    lo_ = 0 if lo is None else int(lo)
    hi_ = m * n if hi is None else int(hi)
    flat = out.view(-1)
    flat[lo_:hi_].copy_(W.detach().reshape(-1)[lo_:hi_])
    plan = _engine_plan(out, g.detach(), state, weights, spec, mode, lo, hi)
    plan.set_step(lr, 0.0, state.t)
    plan.factor_partials()
    plan.factor_finalize()
    plan.stat_sums()[0].copy_(torch.as_tensor(sumsq, dtype=torch.float64))
    # the normalization uses the stats' own element count, as the reference
    # does (a partial-range count normalizes by that range)
    plan.set_stat_counts([int(count)])
    plan.apply()
    _, mx = plan.status()
    return float(mx[0])


@dataclass
class UpdateReport:
    """engine.py:253-262, filled from the device: the pass times are CUDA
    event intervals on the launching stream (pass 1 = factor finalize +
    feature statistics, pass 2 = apply), `kernel_equivalents` the kernels the
    step launched, `scratch_peak_bytes` the plan's device workspace.  Item
    access (report["max_abs_update"]) is kept for dict-style callers."""

    tensor_name: str
    elements: int
    max_abs_update: float
    stats_pass_s: float
    apply_pass_s: float
    kernel_equivalents: int
    scratch_peak_bytes: int

    def __getitem__(self, key):
        if key == "kernel_launches":
            return self.kernel_equivalents
        return getattr(self, key)


def step_fused(W, g, state: DeviceOptState, weights: LoptWeights, spec=None, lr: float = 1.0,
               workers: int = 1, tracker=None, tensor_name: str = "", mode="strict"):
    """engine.py:713-748: returns (new W tensor, UpdateReport).  The state must
    already be advanced for g."""
    spec = spec or small_fc_lopt_spec()
    _check_step_inputs(W, g, state, weights, spec)
    out = W.detach().clone().contiguous()
    plan = _engine_plan(out, g.detach(), state, weights, spec, mode)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    plan.set_step(lr, 0.0, state.t)
    plan.factor_partials()
    ev[0].record()
    plan.factor_finalize()
    plan.feature_stats()
    ev[1].record()
    plan.apply()
    ev[2].record()
    st, mx = plan.status()
    ev[2].synchronize()
    if st[0] & _lib.LOPT_STATUS_NONFINITE_PARAM:
        raise UpdateOverflowError(f"non-finite parameters after fused step {tensor_name!r}")
    report = UpdateReport(tensor_name=tensor_name, elements=W.numel(),
                          max_abs_update=float(mx[0]),
                          stats_pass_s=ev[0].elapsed_time(ev[1]) / 1e3,
                          apply_pass_s=ev[1].elapsed_time(ev[2]) / 1e3,
                          kernel_equivalents=plan.launches_last_step(),
                          scratch_peak_bytes=plan.ws_bytes)
    return out, report


def step_naive(W, g, state: DeviceOptState, weights: LoptWeights, spec=None, lr: float = 1.0,
               tracker=None, tensor_name: str = ""):
    """engine.py:751-826, the reference's non-bitwise class: it materializes
    the features and runs the MLP as a blocked BLAS product, so it agrees with
    step_fused only to the cross-path tolerance 1e-5 (1 + |W|)
    (test_engine.py:262-275).  The device counterpart is the tensor-core
    (fast) path: the same features, the MLP contracted on tcgen05 with an fp16
    two-term split, equally within that tolerance of the fused result."""
    return step_fused(W, g, state, weights, spec, lr, tracker=tracker, tensor_name=tensor_name,
                      mode="fast")
