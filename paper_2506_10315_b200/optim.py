"""torch.optim front end: the drop-in for the reference's optimizer facade.

Mirrors pkg/src/lopt/optim.py:104-180 (OptimizerHandle + opt_step) behind the
torch.optim.Optimizer surface PyLO exposes (PAPER.md:586-601:
`VeLO_CUDA(model.parameters())`, `optimizer.step(loss)`):

  * param_groups with per-group `lr` and `weight_decay` (so
    torch.optim.lr_scheduler works), or a reference ScheduleConfig sampled at
    the pre-increment step counter (optim.py:156);
  * per-step order fixed as in opt_step: accumulators advance, the learned
    update is scaled by lr, decoupled decay multiplies by f32(1 - lr*wd) last;
  * state_dict / load_state_dict carry the accumulators {M1,M2,M3,V} (packed
    per element), the row/column factors and the step counter;
  * a non-finite gradient raises OptimError naming the tensor and changes
    nothing (optim.py:160-165, enforced on the device before any write);
    a non-finite updated parameter raises UpdateOverflowError (engine.py:737)
    -- unlike the reference, the in-place device update has then already been
    written (documented in DESIGN.md).

Tensors are stepped through one StepPlan per parameter group; all kernels run
on the current CUDA stream.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .engine import EngineError, Slot, StepPlan, UpdateOverflowError
from .features import spec_by_name
from .schedule import ScheduleConfig, schedule_lr
from .weights import LoptWeights, random_weights


class OptimError(Exception):
    """optim.py:44-45."""


def view_2d(shape) -> tuple:
    """2-D view of a parameter: rank <= 2 as tensors.py:66-100 (0-D -> (1,1),
    1-D -> (n,1)); rank > 2 (rejected by the reference, tensors.py:77-78) drops
    leading 1s while the rank exceeds 2, then flattens to (d0, prod(rest))."""
    shape = tuple(int(s) for s in shape)
    while len(shape) > 2 and shape[0] == 1:
        shape = shape[1:]
    if len(shape) == 0:
        return (1, 1)
    if len(shape) == 1:
        return (shape[0], 1)
    if len(shape) == 2:
        return shape
    return (shape[0], int(np.prod(shape[1:])))


def _flat_host_view(host, params):
    """A 1-D float32 view over `host` when its tensors are consecutive,
    contiguous pieces of one buffer in parameter order (then a tensor group is
    one copy); None otherwise (per-tensor copies)."""
    if not host or any(t.dtype != torch.float32 or not t.is_contiguous() for t in host):
        return None
    st = host[0].untyped_storage()
    base, off = host[0].data_ptr(), 0
    for t, p in zip(host, params):
        if t.untyped_storage().data_ptr() != st.data_ptr() or t.data_ptr() != base + 4 * off:
            return None
        if t.numel() != p.numel():
            return None
        off += t.numel()
    flat = torch.empty(0, dtype=torch.float32).set_(st, host[0].storage_offset(), (off,))
    return flat


class LearnedOptimizer(torch.optim.Optimizer):
    """Per-parameter MLP learned optimizer (small_fc_lopt / VeLO-MLP features).

    Args:
        params: iterable of float32 CUDA parameters or param-group dicts.
        lr: learning rate scaling the learned update (reference default 1.0).
        weight_decay: decoupled decay coefficient (optim.py:92-101).
        feature_set: "small_fc_lopt" (39 features) or "velo_mlp" (29).
        weights: LoptWeights; default random_weights(d_feat, seed=weights_seed).
        schedule: optional reference ScheduleConfig; when given it overrides
            group lr with schedule_lr(schedule, T) at the pre-increment T.
        mode: "fast" (the default: tensor-core MLP within the fp32 tolerance
            of the reference, states bitwise) or "strict" (every output
            bitwise the reference's; about 4x slower).
        check_errors: synchronize after each step to raise OptimError /
            UpdateOverflowError like the reference; False keeps steps async
            (call `check()` to surface errors later).
    """

    def __init__(self, params, lr: float = 1.0, weight_decay: float = 0.0, *,
                 feature_set: str = "small_fc_lopt", weights: LoptWeights | None = None,
                 weights_seed: int = 0, schedule: ScheduleConfig | None = None,
                 mode: str = "fast", check_errors: bool = True):
        if lr < 0:
            raise ValueError(f"invalid learning rate {lr}")
        if weight_decay < 0:
            raise ValueError("negative weight decay")
        if mode not in ("fast", "strict"):
            raise ValueError(f"unknown mode {mode!r}")
        super().__init__(params, dict(lr=lr, weight_decay=weight_decay))
        self.spec = spec_by_name(feature_set)
        self.lopt_weights = weights or random_weights(self.spec.d_feat, seed=weights_seed)
        if self.lopt_weights.input_dim != self.spec.d_feat:
            raise OptimError(f"MLP input dim {self.lopt_weights.input_dim} does not match "
                             f"feature set ({self.spec.d_feat} columns)")
        self.schedule = schedule
        self.mode = mode
        self.check_errors = check_errors
        self.T = 0
        self.last_loss = None
        self._plans: dict[int, tuple] = {}
        for group in self.param_groups:
            for p in group["params"]:
                if p.dtype != torch.float32:
                    raise TypeError("the learned-optimizer step is float32 (ParamTensor, "
                                    "tensors.py:66)")

    # -- state -------------------------------------------------------------
    def _init_state(self, p):
        st = self.state[p]
        if "quad" not in st:
            m, n = view_2d(p.shape)
            st["quad"] = torch.zeros(m * n, 4, device=p.device, dtype=torch.float32)
            st["row_factors"] = torch.zeros(3, m, device=p.device, dtype=torch.float32)
            st["col_factors"] = torch.zeros(3, n, device=p.device, dtype=torch.float32)
            st["step"] = self.T
        return st

    def _slot(self, p, weight_slot=0) -> Slot:
        if not p.is_cuda or p.grad is None or not p.grad.is_cuda:
            raise TypeError("parameters and gradients must be CUDA tensors (the step runs "
                            "on the device; use step_host for host-resident buffers)")
        st = self._init_state(p)
        m, n = view_2d(p.shape)
        if not p.is_contiguous():
            raise TypeError("parameters must be contiguous")
        g = p.grad
        if g.dtype != torch.float32:
            raise TypeError("gradients must be float32")
        if not g.is_contiguous():
            g = p.grad = g.contiguous()
        return Slot(theta=p.data.view(-1), grad=g.view(-1), state=st["quad"],
                    r=st["row_factors"], c=st["col_factors"], m=m, n=n, weight_slot=weight_slot)

    def _weights_for_group(self, gi, params):
        return self.lopt_weights, [0] * len(params)

    def _plan_for_group(self, gi, params):
        """The group's StepPlan.  Steady state costs one pointer comparison per
        tensor: the plan (and its captured graph) is reused while the same
        parameters carry gradients at the same addresses; moved tensors are
        re-pointed (lopt_rebind_tensors), a different parameter set builds a
        new plan."""
        key = tuple(map(id, params))
        cached = self._plans.get(gi)
        if cached is not None and cached[0] == key:
            _, plan, ptrs = cached
            try:
                now = [(p.data_ptr(), p.grad.data_ptr()) for p in params]
            except AttributeError:
                now = None
            if now == ptrs:
                return plan
        weights, slots_idx = self._weights_for_group(gi, params)
        slots = [self._slot(p, k) for p, k in zip(params, slots_idx)]
        ptrs = [(s.theta.data_ptr(), s.grad.data_ptr()) for s in slots]
        if cached is None or cached[0] != key:
            plan = StepPlan(slots, self.spec, weights, mode=self.mode)
            plan.loss_src = self
            if getattr(self, "_peer_deltas", None):
                plan.set_peers(self._peer_deltas)
        else:
            plan = cached[1]
            plan.rebind(slots)
        self._plans[gi] = (key, plan, ptrs)
        return plan

    # -- step --------------------------------------------------------------
    @torch.no_grad()
    def step(self, closure=None, loss=None):
        """optim.py:144-180.  `loss` is accepted (PyLO's step(loss) signature)
        and recorded; the VeLO subclass feeds it to its hypernetwork."""
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        self.last_loss = None if loss is None else float(loss)
        lr_sched = schedule_lr(self.schedule, self.T) if self.schedule is not None else None
        launched = []
        for gi, group in enumerate(self.param_groups):
            params = [p for p in group["params"] if p.grad is not None]
            if not params:
                continue
            lr = lr_sched if lr_sched is not None else group["lr"]
            plan = self._plan_for_group(gi, params)
            self._run_plan(plan, lr, group["weight_decay"], self.T + 1, gi, params)
            launched.append((plan, params))
        self._pending = launched
        self._last = launched
        if self.check_errors:
            self.check()   # raises before the counter moves, like opt_step
        self.T += 1
        return loss

    # VeLO hypernetwork loss inputs (log loss, EMA), passed with the step
    # scalars of every plan (lopt_step_args.loss_features); unused otherwise
    loss_features = (0.0, 0.0)

    # Hook run after the feature statistics are final and before phase 2
    # (VeLO's hypernetwork mixes the per-tensor MLPs there); None = no hook.
    _after_stats = None

    # optional list collecting (phase, start_event, end_event) per step; the
    # benchmark uses it to time the dominant kernel on the launching stream
    phase_events = None

    def _timed(self, name, fn):
        if self.phase_events is None:
            fn()
            return
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        self.phase_events.append((name, a, b))

    # False: every step launches its kernels one by one (lopt_step) instead of
    # replaying the plan's captured CUDA graph (lopt_graph_step)
    use_graph = True

    def _single_call(self, gi, plan, params) -> bool:
        """True if the whole step of this plan is one C call (VeLO registers
        its hypernetwork on the plan here)."""
        return self._after_stats is None

    def _run_plan(self, plan, lr, weight_decay, t, gi, params):
        if self._single_call(gi, plan, params):
            if self.phase_events is not None:
                # phase events recorded by the C step itself (inside the
                # captured graph when use_graph), so the phase times come from
                # the very steps being measured
                ev = plan.step_timed(lr, weight_decay, t, graph=self.use_graph)
                names = ("factors", "stats", "hypernet", "apply")
                for k, name in enumerate(names):
                    if name != "hypernet" or self._after_stats is not None:
                        self.phase_events.append((name, ev[k], ev[k + 1]))
                return
            plan.clear_phase_events()
            # one C call: all phases (from the captured graph after the first)
            if self.use_graph:
                plan.graph_step(lr, weight_decay, t)
            else:
                plan.step(lr, weight_decay, t)
            return
        plan.set_step(lr, weight_decay, t)
        self._timed("factors", lambda: (plan.factor_partials(), plan.factor_finalize()))
        self._timed("stats", plan.feature_stats)
        if self._after_stats is not None:
            self._timed("hypernet", lambda: self._after_stats(gi, plan, params))
        self._timed("apply", plan.apply)

    def plans(self):
        """The StepPlans of the parameter groups (one per group)."""
        return [entry[1] for entry in self._plans.values()]

    def set_peer_copies(self, deltas):
        """Fused parameter replication (fast mode): the apply pass also stores
        every updated parameter at these byte offsets from its local address
        -- peer GPUs' parameter arenas mapped into this process.  Used by the
        sharded optimizer's NVLink gather; [] disables it."""
        if deltas and self.mode != "fast":
            raise OptimError("peer copies need mode='fast'")
        self._peer_deltas = [int(d) for d in deltas]
        for _, plan, _ in self._plans.values():
            plan.set_peers(self._peer_deltas)

    # -- host-buffer step (offload) ------------------------------------------
    @torch.no_grad()
    def step_host(self, host_grads, host_params=None, *, chunks: int = 8):
        """One step with the gradients in (pinned) host memory and, if given,
        the updated parameters copied back into `host_params` -- the call a
        host-resident caller of the reference makes (opt_step with NumPy
        arrays), served from the device.

        The tensors are cut into `chunks` groups of about equal size, each with
        its own plan; the gradient upload of group k+1 (H2D engine) and the
        parameter download of group k-1 (D2H engine) overlap the device step
        of group k, so the step costs about one PCIe transfer instead of two
        plus the compute.  Semantics per group are those of step(); a
        non-finite gradient aborts its group (groups already stepped stay
        committed -- documented difference to the all-or-nothing opt_step).
        Returns after enqueueing; host_params are valid after a device sync.

        On the first call (and whenever a parameter was moved since) the
        parameters and their gradients are re-homed into two device arenas:
        `p.data` / `p.grad` become views of flat buffers in parameter order.
        When `host_grads` / `host_params` are consecutive views of one pinned
        buffer in the same order, every group crosses PCIe as one copy.  Two
        gradient arenas alternate between calls, so a call's uploads overlap
        the previous call's last groups; `p.grad` views the first arena.
        """
        params = [p for g in self.param_groups for p in g["params"]]
        if len(self.param_groups) != 1:
            raise OptimError("step_host supports one parameter group")
        # NumPy arrays (the reference's calling convention) are wrapped without
        # a copy; pinned torch tensors give asynchronous transfers
        host_grads = [torch.from_numpy(np.ascontiguousarray(g, dtype=np.float32))
                      if isinstance(g, np.ndarray) else g for g in host_grads]
        if host_params is not None:
            for h in host_params:
                if isinstance(h, np.ndarray) and (h.dtype != np.float32 or not h.flags.c_contiguous):
                    raise OptimError("host parameter arrays must be C-contiguous float32")
            host_params = [torch.from_numpy(h) if isinstance(h, np.ndarray) else h
                           for h in host_params]
        if len(host_grads) != len(params):
            raise OptimError(f"got {len(host_grads)} gradients for {len(params)} tensors")
        if host_params is not None and len(host_params) != len(params):
            raise OptimError(f"got {len(host_params)} host parameter buffers for {len(params)}")
        key = (tuple(id(p) for p in params), chunks)
        hs = getattr(self, "_host_step", None)
        if hs is not None and hs["key"] == key:
            # the parameters and gradients must still be the arena views
            pa, ga, offs = hs["parena"].data_ptr(), hs["garena"][0].data_ptr(), hs["offs"]
            if any(p.data.data_ptr() != pa + 4 * offs[k] or p.grad is None
                   or p.grad.data_ptr() != ga + 4 * offs[k] for k, p in enumerate(params)):
                hs = None
        if hs is None or hs["key"] != key:
            # device arenas: parameters and gradients re-homed as views of two
            # flat buffers in parameter order, so a group of tensors moves
            # across PCIe as one contiguous copy (per-tensor copies cost a few
            # microseconds each on the copy engines; ViT-B/16 has 152 tensors)
            total = sum(p.numel() for p in params)
            dev = params[0].device
            parena = torch.empty(total, dtype=torch.float32, device=dev)
            # two gradient arenas, used alternately: the next call's uploads
            # need not wait for this call's last group to finish computing
            garena = [torch.zeros(total, dtype=torch.float32, device=dev) for _ in range(2)]
            offs, off = [], 0
            for p in params:
                n = p.numel()
                parena[off:off + n].copy_(p.data.reshape(-1))
                p.data = parena[off:off + n].view(p.shape)
                p.grad = garena[0][off:off + n].view(p.shape)
                offs.append(off)
                off += n
            offs.append(off)
            groups, cur, acc = [], [], 0
            for k, p in enumerate(params):
                cur.append(k)
                acc += p.numel()
                if acc >= total * (len(groups) + 1) / chunks and len(groups) < chunks - 1:
                    groups.append(cur)
                    cur = []
            if cur:
                groups.append(cur)
            hs = {"key": key, "groups": groups,
                  "plans": [[None] * len(groups), [None] * len(groups)],
                  "ptrs": [{}, {}], "read_done": [None, None], "parity": 0,
                  "h2d": torch.cuda.Stream(), "d2h": torch.cuda.Stream(),
                  "parena": parena, "garena": garena, "offs": offs}
            self._host_step = hs
        offs = hs["offs"]
        hg_flat = _flat_host_view(host_grads, params)
        hp_flat = _flat_host_view(host_params, params) if host_params is not None else None
        group = self.param_groups[0]
        lr = schedule_lr(self.schedule, self.T) if self.schedule is not None else group["lr"]
        wd, t = group["weight_decay"], self.T + 1
        comp = torch.cuda.current_stream()
        h2d, d2h = hs["h2d"], hs["d2h"]
        uploaded = []
        b = hs["parity"]
        hs["parity"] ^= 1
        garena = hs["garena"][b]
        # this buffer was last read by the step before the previous one
        if hs["read_done"][b] is not None:
            h2d.wait_event(hs["read_done"][b])
        else:
            h2d.wait_stream(comp)
        with torch.cuda.stream(h2d):
            for ks in hs["groups"]:
                if hg_flat is not None:
                    o0, o1 = offs[ks[0]], offs[ks[-1] + 1]
                    garena[o0:o1].copy_(hg_flat[o0:o1], non_blocking=True)
                else:
                    for k in ks:
                        garena[offs[k]:offs[k + 1]].copy_(host_grads[k].reshape(-1),
                                                          non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(h2d)
                uploaded.append(ev)
        launched = []
        d2h.wait_stream(comp)
        for gi, ks in enumerate(hs["groups"]):
            comp.wait_event(uploaded[gi])
            ps = [params[k] for k in ks]
            plan = hs["plans"][b][gi]
            hkey = ("host", gi)
            weights, widx = self._weights_for_group(hkey, ps)
            slots = [self._slot(p, w) for p, w in zip(ps, widx)]
            for k, sl in zip(ks, slots):
                sl.grad = garena[offs[k]:offs[k + 1]]
            ptrs = [(sl.theta.data_ptr(), sl.grad.data_ptr()) for sl in slots]
            if plan is None:
                plan = StepPlan(slots, self.spec, weights, mode=self.mode)
                plan.loss_src = self
                hs["plans"][b][gi] = plan
                hs["ptrs"][b][gi] = ptrs
            elif hs["ptrs"][b][gi] != ptrs:
                plan.rebind(slots)
                hs["ptrs"][b][gi] = ptrs
            if self._after_stats is None:
                plan.step(lr, wd, t)
            else:   # VeLO: the per-tensor hypernetwork between phases 1 and 2
                plan.set_step(lr, wd, t)
                plan.factor_partials()
                plan.factor_finalize()
                plan.feature_stats()
                self._after_stats(hkey, plan, ps)
                plan.apply()
            launched.append((plan, ps))
            if host_params is not None:
                done = torch.cuda.Event()
                done.record(comp)
                d2h.wait_event(done)
                with torch.cuda.stream(d2h):
                    if hp_flat is not None:
                        o0, o1 = offs[ks[0]], offs[ks[-1] + 1]
                        hp_flat[o0:o1].copy_(hs["parena"][o0:o1], non_blocking=True)
                    else:
                        for k in ks:
                            host_params[k].view(params[k].shape).copy_(params[k].detach(),
                                                                        non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(comp)              # the last group has read gradient buffer b
        hs["read_done"][b] = ev
        comp.wait_stream(d2h)        # the next step's applies write what these copies read
        self._pending = launched
        self._last = launched
        if self.check_errors:
            self.check()
        self.T += 1
        return None

    def check(self):
        """Surface device-side errors of the last step (synchronizes)."""
        pending, self._pending = getattr(self, "_pending", []), []
        for plan, params in pending:
            st, _ = plan.status()
            for j, s in enumerate(st):
                if s & _lib.LOPT_STATUS_NONFINITE_GRAD:
                    raise OptimError(f"tensor {self._name(params[j])!r}: non-finite gradient")
            for j, s in enumerate(st):
                if s & _lib.LOPT_STATUS_NONFINITE_PARAM:
                    raise UpdateOverflowError(
                        f"non-finite parameters after fused step {self._name(params[j])!r}")

    def _name(self, p):
        for gi, group in enumerate(self.param_groups):
            for k, q in enumerate(group["params"]):
                if q is p:
                    return f"group{gi}.param{k}"
        return "?"

    def max_abs_updates(self):
        """UpdateReport.max_abs_update per stepped tensor of the last step."""
        out = []
        for plan, _ in getattr(self, "_last", []):
            out.extend(plan.status()[1].tolist())
        return out

    # -- checkpointing -------------------------------------------------------
    def state_dict(self):
        for st in self.state.values():   # the per-tensor step counter, kept lazily
            if "quad" in st:
                st["step"] = self.T
        sd = super().state_dict()
        sd["lopt"] = {"T": self.T, "feature_set": self.spec.id.value, "mode": self.mode,
                      "weights": [(w.copy(), b.copy()) for w, b in self.lopt_weights.layers]}
        return sd

    def load_state_dict(self, state_dict):
        extra = state_dict.get("lopt", {})
        if extra.get("feature_set", self.spec.id.value) != self.spec.id.value:
            raise OptimError(f"checkpoint feature set {extra['feature_set']!r}, expected "
                             f"{self.spec.id.value!r}")
        sd = {k: v for k, v in state_dict.items() if k != "lopt"}
        super().load_state_dict(sd)
        for st in self.state.values():
            for k in ("quad", "row_factors", "col_factors"):
                if k in st:
                    st[k] = st[k].to(torch.float32).contiguous()
        self.T = int(extra.get("T", self.T))
        self._plans.clear()
        self._host_step = None   # its plans point at the replaced state tensors


class AdafacLO_CUDA(LearnedOptimizer):
    """small_fc_lopt (the Adafactor-featured per-parameter MLP)."""

    def __init__(self, params, lr: float = 1.0, weight_decay: float = 0.0, **kw):
        kw.setdefault("feature_set", "small_fc_lopt")
        super().__init__(params, lr=lr, weight_decay=weight_decay, **kw)


def opt_step(opt: LearnedOptimizer, grads, loss=None):
    """The reference's functional entry point opt_step(h, grads, loss)
    (optim.py:144-180) over an optimizer: one gradient per parameter in
    parameter order (device tensors), the same count / shape errors, then
    one step."""
    ps = [p for g in opt.param_groups for p in g["params"]]
    if len(grads) != len(ps):
        raise OptimError(f"got {len(grads)} gradients for {len(ps)} tensors")
    for p, g in zip(ps, grads):
        if tuple(g.shape) != tuple(p.shape):
            raise OptimError(f"gradient {tuple(g.shape)} vs param {tuple(p.shape)}")
        p.grad = g
    return opt.step(loss=loss)
