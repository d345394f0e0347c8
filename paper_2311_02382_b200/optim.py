"""Optimizers over the engine's flat fp32 parameter / gradient buffers.

Mirrors the reference's optimizer API (seqpar.optim, optim.py:18-68;
model.sgd_step, model.py:621-623): ``make_update(name, lr)`` returns an
object whose ``step(params, grads)`` updates ``params`` in place with one
fused kernel (lss_sgd_update / lss_adam_update).  As in the reference, every
worker owns its optimizer and its state never crosses worker boundaries.
"""

from __future__ import annotations

import torch

from . import kernels as K

OPTIMIZERS = ("sgd", "adam")


class SGD:
    """model.sgd_step: w - lr * g."""

    def __init__(self, lr: float):
        self.lr = float(lr)

    def step(self, params: torch.Tensor, grads: torch.Tensor) -> None:
        K.sgd_update(params, grads, self.lr)


class Adam:
    """optim.adam_step: bias-corrected Adam (beta1 0.9, beta2 0.999, eps 1e-8)."""

    def __init__(self, lr: float, beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8):
        self.lr, self.beta1, self.beta2, self.eps = float(lr), beta1, beta2, eps
        self.t = 0
        self.m = self.v = None

    def step(self, params: torch.Tensor, grads: torch.Tensor) -> None:
        if self.m is None:
            self.m, self.v = torch.zeros_like(params), torch.zeros_like(params)
        self.t += 1
        K.adam_update(params, grads, self.m, self.v, lr=self.lr, step=self.t, beta1=self.beta1,
                      beta2=self.beta2, eps=self.eps)


def make_update(name: str, lr: float):
    """optim.make_update (optim.py:56-68)."""
    if name == "sgd":
        return SGD(lr)
    if name == "adam":
        return Adam(lr)
    raise ValueError(f"unknown optimizer {name!r}, expected one of {OPTIMIZERS}")
