"""The reference's hand-designed baseline optimizers on the device
(SURVEY.md section 8(f) rank 4): same functional signatures and conventions as
pkg/src/lopt/optim.py:187-217, so the learned step's overhead is compared like
for like (bench.py `context`).  CUDA tensors are updated in place and returned.

    adam_step       optim.py:187-198   bias-corrected Adam (bitwise the reference)
    adafactor_step  optim.py:201-217   factored second moment, plain step size
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib

F32 = np.float32


def _cuda_f32(name, x):
    if not isinstance(x, torch.Tensor) or not x.is_cuda or x.dtype != torch.float32:
        raise TypeError(f"{name} must be a float32 CUDA tensor")
    if not x.is_contiguous():
        raise TypeError(f"{name} must be contiguous")
    return x


def adam_step(theta, g, m, v, beta1=0.9, beta2=0.999, lr=1e-3, eps=1e-8, t=1):
    """optim.py:187-198, in place on (theta, m, v); returns them."""
    if t < 1:
        raise ValueError("Adam step count starts at 1")
    for nm, x in (("theta", theta), ("g", g), ("m", m), ("v", v)):
        _cuda_f32(nm, x)
        if x.shape != theta.shape:
            raise ValueError(f"{nm} shape {tuple(x.shape)} != theta {tuple(theta.shape)}")
    b1, b2 = F32(beta1), F32(beta2)
    # the reference's numpy f32 scalars (b ** F32(t) is numpy's f32 power)
    sc = np.array([b1, F32(1.0) - b1, b2, F32(1.0) - b2, F32(1.0) - b1 ** F32(t),
                   F32(1.0) - b2 ** F32(t), F32(lr), F32(eps)], dtype=F32)
    L = _lib.require_cuda()
    _lib.check(L.lopt_adam_step(theta.data_ptr(), g.data_ptr(), m.data_ptr(), v.data_ptr(),
                                theta.numel(), sc.ctypes.data,
                                torch.cuda.current_stream().cuda_stream), "adam_step")
    return theta, m, v


_scratch = {}


def adafactor_step(theta, g, r, c, beta=0.999, lr=1e-3, eps=1e-30):
    """optim.py:201-217 on a 2-D (rows, cols) theta, in place on (theta, r, c);
    returns them."""
    for nm, x in (("theta", theta), ("g", g), ("r", r), ("c", c)):
        _cuda_f32(nm, x)
    if theta.dim() != 2 or g.shape != theta.shape:
        raise ValueError("adafactor_step takes 2-D theta and g of the same shape")
    rows, cols = theta.shape
    if rows == 0 or cols == 0:
        raise ValueError("adafactor factors undefined for empty tensors")   # state.py:102-103
    if r.shape != (rows,) or c.shape != (cols,):
        raise ValueError(f"factor shapes {tuple(r.shape)}/{tuple(c.shape)} do not match "
                         f"gradient {tuple(g.shape)}")
    b = F32(beta)
    sc = np.array([b, F32(1.0) - b, F32(lr), F32(eps)], dtype=F32)
    L = _lib.require_cuda()
    need = int(L.lopt_adafactor_scratch_bytes(rows, cols))
    dev = theta.device
    buf = _scratch.get(dev)
    if buf is None or buf.numel() * 8 < need:
        buf = _scratch[dev] = torch.empty((need + 7) // 8, dtype=torch.float64, device=dev)
    _lib.check(L.lopt_adafactor_step(theta.data_ptr(), g.data_ptr(), r.data_ptr(), c.data_ptr(),
                                     rows, cols, sc.ctypes.data, buf.data_ptr(),
                                     torch.cuda.current_stream().cuda_stream), "adafactor_step")
    return theta, r, c
