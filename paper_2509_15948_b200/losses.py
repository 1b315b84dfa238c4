"""Audio loss API (mg/losses.py) on the device.

``mrstft(y_hat, target, cfg)`` is the multi-resolution A-weighted log-mel +
spectral-convergence distance; ``target`` is a (2, Ls) signal or a
``PreparedTarget`` whose spectra live on the device (computed once per eval
segment, as the reference caches them, mg/losses.py:111-140).  It is a torch
autograd op whose backward is ``mgb_mrstft_backward``.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from .common import SAMPLE_RATE
from .engine import F32, F64, LossPlan, ensure_device, ptr
from .schedule import LengthMismatch

LOG_EPS = 1e-7
NORM_EPS = 1e-12


@dataclass(frozen=True)
class LossConfig:
    fft_sizes: tuple = (512, 1024, 4096)
    mel_bins: int = 96
    weight_lr: float = 0.5
    weight_mid: float = 0.25
    weight_side: float = 0.25
    gain_staging_weight: float = 1e-3
    mel_fmax: float = 15_000.0
    a_weighting: bool = True
    sample_rate: int = SAMPLE_RATE

    def __post_init__(self):
        total = self.weight_lr + self.weight_mid + self.weight_side
        if abs(total - 1.0) > 1e-12:
            raise ValueError(f"channel weights sum to {total}, expected 1.0")
        if any(s <= 0 for s in self.fft_sizes) or self.mel_bins <= 0:
            raise ValueError("sizes must be positive")

    def hop(self, n_fft):
        return n_fft // 4


class PreparedTarget:
    """Target spectra resident on the device (mg/losses.py:111-140)."""

    def __init__(self, y, cfg: LossConfig = LossConfig(), device=None):
        t = y if torch.is_tensor(y) else torch.as_tensor(np.asarray(y))
        dev = ensure_device(device or (t.device if t.is_cuda else "cuda"))
        self.signal = t.to(device=dev, dtype=F32).contiguous()
        self.length = self.signal.shape[-1]
        self.cfg = cfg
        self.plan = LossPlan(cfg, self.length, dev)
        self.plan.target(ptr(self.signal, 0), ptr(self.signal, self.length))


def prepare_target(y, cfg: LossConfig = LossConfig()):
    return PreparedTarget(y, cfg)


class _MRSTFTFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, y_hat, prepared):
        plan = prepared.plan
        y = y_hat.contiguous()
        Ls = y.shape[-1]
        plan.forward(ptr(y, 0), ptr(y, Ls))
        ctx.save_for_backward(y)
        ctx.prepared = prepared
        return plan.loss.clone()

    @staticmethod
    def backward(ctx, g):
        (y,) = ctx.saved_tensors
        plan = ctx.prepared.plan
        Ls = y.shape[-1]
        gy = torch.empty_like(y)
        plan.backward(ptr(y, 0), ptr(y, Ls), ptr(gy, 0), ptr(gy, Ls))
        return gy * g.to(F32), None


def mrstft(y_hat, target, cfg: LossConfig = LossConfig()):
    yt = y_hat if torch.is_tensor(y_hat) else torch.as_tensor(np.asarray(y_hat))
    if not yt.is_cuda:
        yt = yt.to(ensure_device("cuda"))
    yt = yt.to(F32)
    if not isinstance(target, PreparedTarget):
        target = PreparedTarget(target, cfg, yt.device)
    if yt.shape[-1] != target.length:
        raise LengthMismatch(f"estimate length {yt.shape[-1]} != target {target.length}")
    return _MRSTFTFn.apply(yt, target)


def sparsity_loss(weights):
    """l1 norm of the dry/wet weights (mg/losses.py:181-183)."""
    return torch.sum(torch.as_tensor(weights, dtype=F64))
