"""VeLO: the VELO_MLP per-element optimizer driven by a per-tensor LSTM
hypernetwork that mixes a bank of per-element MLPs.

The reference ships only the per-element half (the 29-column VELO_MLP feature
set with one global MLP, features.py:24-28) and lists the hypernetwork as out
of scope.  This module adds the build-defined hypernetwork of
SURVEY.md section 8(a) row 15 (definition and numpy restatement:
oracle/velo_lstm.py; device kernel: csrc/lopt_velo.cu):

    per tensor and step: LSTM over [log E[f^2] (29) | tanh(t/x) (11) | loss (2)]
    -> softmax mixing weights over K bank MLPs -> this tensor's MLP.

With a bank of one MLP the mixture is that MLP, so VeLO_CUDA reduces exactly
to the reference's VELO_MLP step (the parity anchor for the per-element path).
PyLO's API needs the loss at every step: `optimizer.step(loss)`.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .optim import LearnedOptimizer, OptimError
from .weights import LoptWeights, random_weights, unpack

F32 = np.float32
N_IN = 42


class VeLOHyperNet:
    """Hypernetwork parameters (LSTM + mixing head) and the MLP bank."""

    def __init__(self, hidden: int = 16, bank_size: int = 4, seed: int = 0,
                 hyper: np.ndarray | None = None, bank: list | None = None):
        if not 1 <= hidden <= 64 or not 1 <= bank_size <= 16:
            raise ValueError("hidden must be in [1, 64] and bank_size in [1, 16]")
        self.H, self.K = hidden, bank_size
        n = 4 * hidden * N_IN + 4 * hidden * hidden + 4 * hidden + bank_size * hidden + bank_size
        if hyper is None:
            rng = np.random.default_rng(seed)
            hyper = (rng.standard_normal(n) * 0.1).astype(F32)
            off = 4 * hidden * N_IN + 4 * hidden * hidden
            hyper[off + hidden: off + 2 * hidden] = F32(1.0)   # forget-gate bias
        self.hyper = np.ascontiguousarray(hyper, F32)
        if self.hyper.size != n:
            raise ValueError(f"hypernetwork has {self.hyper.size} parameters, expected {n}")
        if bank is None:
            bank = [random_weights(29, seed=seed * 1000 + k) for k in range(bank_size)]
        if len(bank) != bank_size:
            raise ValueError("bank size mismatch")
        for w in bank:
            if w.input_dim != 29:
                raise ValueError("VeLO bank MLPs take the 29 VELO_MLP features")
        self.bank = bank

    def packed_bank(self) -> np.ndarray:
        return np.stack([w.packed() for w in self.bank]).astype(F32)


class _VeLOMixin:
    """Adds the hypernetwork pass between phase 1 and phase 2."""

    def _velo_init(self, hypernet: VeLOHyperNet | None):
        self.hypernet = hypernet or VeLOHyperNet()
        dev = self.param_groups[0]["params"][0].device
        self._hyper_dev = torch.from_numpy(self.hypernet.hyper).to(dev)
        self._bank_dev = torch.from_numpy(self.hypernet.packed_bank()).to(dev)
        self._loss_ema = None
        self._lstm = {}

    def _weights_for_group(self, gi, params):
        # one weight slot per tensor, filled on the device by the hypernetwork
        return [self.hypernet.bank[0]] * len(params), list(range(len(params)))

    def _lstm_state(self, gi, params):
        key = tuple(id(p) for p in params)
        st, old_key = self._lstm.get(gi, (None, None))
        if st is None or old_key != key:
            # one contiguous [tensors x 2H] block per group for the kernel;
            # rows start from the tensors' current LSTM state (a resumed or
            # regrouped optimizer continues where it was)
            dev = params[0].device
            st = torch.zeros(len(params), 2 * self.hypernet.H, dtype=torch.float32, device=dev)
            for j, p in enumerate(params):
                prev = self.state[p].get("lstm")
                if prev is not None:
                    st[j].copy_(prev.to(device=dev, dtype=torch.float32).reshape(-1))
                self.state[p]["lstm"] = st[j]
            # keyed by the parameters' identities: if the set of tensors with
            # gradients changes, each tensor keeps its own row
            self._lstm[gi] = (st, key)
        return st

    def state_dict(self):
        sd = super().state_dict()
        sd["velo"] = {"loss_ema": self._loss_ema}
        return sd

    def load_state_dict(self, state_dict):
        extra = state_dict.get("velo", {})
        super().load_state_dict({k: v for k, v in state_dict.items() if k != "velo"})
        self._lstm = {}   # rebuilt from the loaded per-tensor rows on the next step
        self._loss_ema = extra.get("loss_ema", self._loss_ema)

    def _set_loss(self, loss):
        if loss is None:
            raise OptimError("VeLO needs the loss: call optimizer.step(loss) (PAPER.md:600)")
        lv = math.log(max(float(loss), 1e-8))
        # kept so that a step that changes nothing (non-finite gradient,
        # optim.py:160-165) also leaves the loss EMA where it was (check())
        self._loss_ema_prev = self._loss_ema
        self._loss_ema = lv if self._loss_ema is None else 0.9 * self._loss_ema + 0.1 * lv
        # the hypernetwork reads them from the step scalars (lopt_step_args):
        # no upload, nothing to synchronize
        self.loss_features = (lv, self._loss_ema)

    def check(self):
        """LearnedOptimizer.check; an aborted step (OptimError: non-finite
        gradient) also rolls the loss EMA back -- on the device the
        hypernetwork kernel skipped the LSTM update (lopt_velo.cu)."""
        try:
            super().check()
        except OptimError:
            if hasattr(self, "_loss_ema_prev"):
                self._loss_ema = self._loss_ema_prev
            raise

    def _single_call(self, gi, plan, params) -> bool:
        """One-device step: the hypernetwork is registered on the plan and
        runs inside lopt_step / the captured graph."""
        st = self._lstm_state(gi, params)
        mix = getattr(self, "_mix_out", None)
        key = (self._hyper_dev.data_ptr(), st.data_ptr(), self._bank_dev.data_ptr(),
               None, mix.data_ptr() if mix is not None else None)
        if plan._velo_key != key:
            plan.set_velo(self._hyper_dev, st, self._bank_dev, None, self.hypernet.H,
                          self.hypernet.K, mix)
        return True

    def _after_stats(self, gi, plan, params):
        st = self._lstm_state(gi, params)
        mix = getattr(self, "_mix_out", None)
        _lib.check(plan.L.lopt_velo_mix(
            plan.h, self._hyper_dev.data_ptr(), st.data_ptr(), self._bank_dev.data_ptr(),
            None, self.hypernet.H, self.hypernet.K,
            mix.data_ptr() if mix is not None else None,
            torch.cuda.current_stream().cuda_stream), "velo_mix")


class VeLO_CUDA(_VeLOMixin, LearnedOptimizer):
    """PyLO's `VeLO_CUDA(model.parameters())` surface: VELO_MLP features, a
    per-tensor MLP mixed by the LSTM hypernetwork, `step(loss)`."""

    def __init__(self, params, lr: float = 1.0, weight_decay: float = 0.0, *,
                 hypernet: VeLOHyperNet | None = None, **kw):
        kw.pop("feature_set", None)
        hn = hypernet or VeLOHyperNet()
        super().__init__(params, lr=lr, weight_decay=weight_decay, feature_set="velo_mlp",
                         weights=hn.bank[0], **kw)
        self._velo_init(hn)

    def step(self, closure=None, loss=None):
        if closure is not None:
            with torch.enable_grad():
                loss = closure()
        self._set_loss(loss)
        return super().step(loss=loss)

    def step_host(self, host_grads, host_params=None, *, chunks: int = 8, loss=None):
        """LearnedOptimizer.step_host with the loss VeLO's hypernetwork needs;
        each tensor group runs the hypernetwork between its phases 1 and 2
        (per-tensor LSTM state kept per group: do not alternate with step())."""
        self._set_loss(loss)
        return super().step_host(host_grads, host_params, chunks=chunks)
