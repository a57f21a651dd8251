"""Composite training objective and its analytic gradients (B200).

Drop-in for the reference's ``splatct.loss`` (loss.py:1-253).  L1 and SSIM
run in the fused projection-loss kernels (csrc/loss.cu), TV in the
TV-fused adjoint kernel (csrc/proj.cu) with an empty projector, so the
standalone API evaluates exactly the code the training iteration runs.
Values are float64 like the reference; gradients are returned as float64
arrays holding the kernels' float32 results (the training loop quantises
them to float32 at the same point, optim.py:368,371).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .core import Sinogram, ValidationError, VolumeGrid

__all__ = ["LossWeights", "WEIGHT_PRESETS", "l1_loss", "ssim_loss", "ssim_value", "total_loss",
           "total_loss_detailed", "tv_loss"]


@dataclass(frozen=True)
class LossWeights:
    """Weights of the L1, SSIM and TV terms (loss.py:35-48)."""

    lambda1: float = 0.6
    lambda2: float = 0.2
    lambda3: float = 1.0

    def __post_init__(self):
        ws = (self.lambda1, self.lambda2, self.lambda3)
        if any(v < 0 for v in ws):
            raise ValidationError(f"loss weights must be non-negative, got {ws}")
        if not any(v > 0 for v in ws):
            raise ValidationError("at least one loss weight must be positive")


WEIGHT_PRESETS = {
    "l1": LossWeights(1.0, 0.0, 0.0),
    "l1+ssim": LossWeights(0.8, 0.2, 0.0),
    "l1+ssim+tv": LossWeights(0.6, 0.2, 1.0),
}


def _match_dims(pred: Sinogram, ref: Sinogram) -> None:
    if pred.dims != ref.dims:
        raise ValidationError(f"sinogram dims differ: {pred.dims} vs {ref.dims}")


def ssim_valid_count(m: int, n: int) -> int:
    """Number of fully covered window positions (loss.py:104-109 windows)."""
    kr, kc = min(11, m), min(11, n)
    kr -= 1 - kr % 2
    kc -= 1 - kc % 2
    return (m - kr + 1) * (n - kc + 1)


def _fused(pred_v: np.ndarray, ref_v: np.ndarray, l1w: float, ssw: float, lmax=None):
    """Run the fused kernel on host arrays (m, n, p): (sums, grad (m,n,p) f64)."""
    dev = D.require_cuda()
    m, n, p = pred_v.shape
    x = D.sino_to_device(pred_v, dev)
    y = D.sino_to_device(ref_v, dev)
    if lmax is None:
        lmax = D.sino_max(y)
    plan = D.LossPlan(m, n, p, dev)
    g = torch.empty_like(x)
    sums = torch.zeros(3, dtype=torch.float64, device=dev)
    plan.fused(x, y, lmax, l1w, ssw, float(m * n * p), float(p), g, sums)
    return sums.cpu().numpy(), g.double().cpu().numpy(), plan.valid


def l1_loss(pred: Sinogram, ref: Sinogram):
    """Mean absolute error; subgradient sign/count (loss.py:64-74)."""
    _match_dims(pred, ref)
    sums, g, _ = _fused(pred.views, ref.views, 1.0, 0.0)
    return float(sums[0] / pred.data.size), g


def ssim_loss(pred: Sinogram, ref: Sinogram):
    """1 - mean SSIM over slices, and its gradient (loss.py:159-180)."""
    _match_dims(pred, ref)
    sums, g, val = _fused(pred.views, ref.views, 0.0, 1.0)
    p = pred.dims[2]
    return 1.0 - float(sums[1] / val / p), g


def ssim_value(x, y, max_val: float | None = None) -> float:
    """Mean SSIM of a 2D image pair (loss.py:144-156)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    if x.shape != y.shape:
        raise ValidationError(f"image shapes differ: {x.shape} vs {y.shape}")
    lmax = float(np.max(y)) if max_val is None else float(max_val)
    if lmax <= 0:
        lmax = 1.0
    sums, _, val = _fused(x[:, :, None].astype(np.float32), y[:, :, None].astype(np.float32),
                          0.0, 1.0, lmax=lmax)
    return float(sums[1] / val)


def tv_loss(vol: VolumeGrid):
    """Anisotropic TV with zero-flux boundaries (loss.py:183-207)."""
    dev = D.require_cuda()
    w, h, c = vol.dims
    v = D.zyx_to_yxz(vol.zyx, dev)
    op = D.tv_operator(w, h, dev)
    count = float(w * h * c)
    part = torch.empty(w * h, dtype=torch.float64, device=dev)
    zero = torch.zeros((1, 1, c), dtype=torch.float32, device=dev)
    out = torch.empty_like(v)
    op.adjoint(zero, out, vol=v, lambda_tv=1.0, tv_count=count, tv_partial=part)
    tot = torch.empty(1, dtype=torch.float64, device=dev)
    D.reduce_sum(part, tot)
    return float(tot.item()) / count, D.yxz_to_zyx(out).astype(np.float64)


def total_loss_detailed(pred: Sinogram, ref: Sinogram, vol: VolumeGrid, weights: LossWeights):
    """Weighted sum plus unweighted parts; zero-weight terms -> NaN (loss.py:210-239)."""
    _match_dims(pred, ref)
    value = 0.0
    parts = {"l1": float("nan"), "ssim": float("nan"), "tv": float("nan")}
    grad_vol = np.zeros(vol.zyx.shape)
    if weights.lambda1 > 0 or weights.lambda2 > 0:
        sums, grad_pred, val = _fused(pred.views, ref.views, weights.lambda1, weights.lambda2)
    else:
        grad_pred = np.zeros(pred.views.shape)
    m, n, p = pred.dims
    if weights.lambda1 > 0:
        parts["l1"] = float(sums[0] / (m * n * p))
        value += weights.lambda1 * parts["l1"]
    if weights.lambda2 > 0:
        parts["ssim"] = 1.0 - float(sums[1] / val / p)
        value += weights.lambda2 * parts["ssim"]
    if weights.lambda3 > 0:
        tv, g = tv_loss(vol)
        parts["tv"] = tv
        value += weights.lambda3 * tv
        grad_vol = weights.lambda3 * g
    return value, grad_pred, grad_vol, parts


def total_loss(pred: Sinogram, ref: Sinogram, vol: VolumeGrid, weights: LossWeights):
    """(value, grad wrt pred (m,n,p), grad wrt vol (c,h,w)) (loss.py:242-253)."""
    value, gp, gv, _ = total_loss_detailed(pred, ref, vol, weights)
    return value, gp, gv
