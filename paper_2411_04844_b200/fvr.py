"""Fast Volume Reconstruction: splat Gaussians onto the voxel grid (B200).

Drop-in for the reference's ``splatct.fvr`` (fvr.py:1-273): same functions,
signatures, validation and warnings; the arithmetic runs in the tiled
sm_100a kernels of csrc/fvr.cu.  ``deterministic`` is accepted for API
compatibility: the device path is always bitwise reproducible (fixed
per-tile Gaussian order, no floating-point atomics).
"""

from __future__ import annotations

import warnings
from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from .core import (
    BoxConfig,
    GaussianCloud,
    OffsetGrid,
    ParamGradients,
    ValidationError,
    VolumeGrid,
    make_offset_grid,
    require_valid_cloud,
)

__all__ = [
    "DenseBudgetError",
    "FvrWorkspace",
    "backward",
    "reconstruct",
    "reconstruct_direct",
    "reconstruct_nodecomp",
    "sq_distance_decomposed",
    "sq_distance_direct",
    "truncation_bound",
]

DEFAULT_DENSE_BUDGET = 200_000_000


class DenseBudgetError(RuntimeError):
    """Dense evaluation would exceed the element budget (fvr.py:54-55)."""


@dataclass(frozen=True)
class FvrWorkspace:
    """Per-box constants: offsets and exact integer b.b (fvr.py:58-76)."""

    box: BoxConfig
    offset_grid: OffsetGrid
    btb: np.ndarray

    @classmethod
    def create(cls, box: BoxConfig) -> "FvrWorkspace":
        g = make_offset_grid(box)
        btb = np.einsum("ij,ij->i", g.offsets, g.offsets).astype(np.float64)
        btb.setflags(write=False)
        return cls(box, g, btb)


def sq_distance_direct(b, dmu, sigma):
    """(b - dmu).(b - dmu) / sigma^2 (fvr.py:79-84)."""
    r = np.asarray(b, np.float64) - np.asarray(dmu, np.float64)
    return np.sum(r * r, axis=-1) / np.asarray(sigma, np.float64) ** 2


def sq_distance_decomposed(b, dmu, sigma):
    """Four-term expansion b.b - b.dmu - dmu.b + dmu.dmu, over sigma^2 (fvr.py:87-101)."""
    b = np.asarray(b, np.float64)
    d = np.asarray(dmu, np.float64)
    terms = (np.sum(b * b, -1), np.sum(b * d, -1), np.sum(d * b, -1), np.sum(d * d, -1))
    return (terms[0] - terms[1] - terms[2] + terms[3]) / np.asarray(sigma, np.float64) ** 2


def truncation_bound(box: BoxConfig, cloud: GaussianCloud, dims=None) -> float:
    """Bound on the value any voxel loses to box confinement (fvr.py:104-120)."""
    halves = list(box.half)
    if dims is not None:
        halves = [hf for hf, side, d in zip(box.half, box.shape, dims) if side < int(d)]
        if not halves:
            return 0.0
    d = min(halves)
    return float(np.sum(cloud.intensity * np.exp(-0.5 * d * d / cloud.sigma ** 2)))


def _check_args(cloud: GaussianCloud, box: BoxConfig, dims):
    """Validation of fvr.py:123-139 (errors and the out-of-volume warning)."""
    require_valid_cloud(cloud)
    w, h, c = (int(v) for v in dims)
    if box.w0 > w or box.h0 > h or box.c0 > c:
        raise ValidationError(f"box {box.shape} exceeds volume dims {(w, h, c)} along some axis")
    if (cloud.mu.min(axis=0) < 0).any() or (cloud.mu.max(axis=0) >= np.array([w, h, c])).any():
        warnings.warn("Gaussian centers outside the volume; their out-of-bounds contributions "
                      "are clipped", RuntimeWarning, stacklevel=3)
    return w, h, c


def reconstruct_device(params: torch.Tensor, box: BoxConfig, dims, plan: D.FvrPlan | None = None,
                       out: torch.Tensor | None = None) -> torch.Tensor:
    """Device-resident splat: params [5,N] f64 -> volume (h, w, c) f32."""
    if plan is None:
        plan = D.FvrPlan(params.shape[1], dims, box.half, 0, params.device)
    if out is None:
        out = plan.new_volume()
    plan.bin(params)
    plan.forward(params, out)
    return out


def reconstruct(cloud: GaussianCloud, box: BoxConfig, dims,
                deterministic: bool = False) -> VolumeGrid:
    """Splat the cloud onto a zero-initialised (w, h, c) grid (fvr.py:148-167)."""
    w, h, c = _check_args(cloud, box, dims)
    dev = D.require_cuda()
    params = D.cloud_to_params(cloud, dev)
    vol = reconstruct_device(params, box, (w, h, c))
    return VolumeGrid.from_zyx(D.yxz_to_zyx(vol))


def reconstruct_nodecomp(cloud: GaussianCloud, box: BoxConfig, dims,
                         deterministic: bool = False) -> VolumeGrid:
    """Splat without the decomposition (fvr.py:170-190 -> _kernels.splat_plain
    :81-129): the same bins, clipping and tile-owned accumulation as
    :func:`reconstruct`, but every box voxel pays its own squared distance and
    exponential -- the comparator the decomposition is measured against."""
    w, h, c = _check_args(cloud, box, dims)
    dev = D.require_cuda()
    params = D.cloud_to_params(cloud, dev)
    plan = D.FvrPlan(params.shape[1], (w, h, c), box.half, 0, dev)
    out = plan.new_volume()
    plan.bin(params)
    plan.forward_plain(params, out)
    return VolumeGrid.from_zyx(D.yxz_to_zyx(out))


def reconstruct_direct(cloud: GaussianCloud, dims, budget: int = DEFAULT_DENSE_BUDGET) -> VolumeGrid:
    """Unconfined dense sum over every voxel (fvr.py:193-224).

    A brute-force oracle in the reference; evaluated here on the device as
    a box covering the whole grid (every Gaussian reaches every voxel).
    """
    require_valid_cloud(cloud)
    w, h, c = (int(v) for v in dims)
    if cloud.n * w * h * c > budget:
        raise DenseBudgetError(f"dense evaluation needs {cloud.n * w * h * c} element visits, "
                               f"over the budget of {budget}")
    dev = D.require_cuda()
    # a box of half-width max(dim) around floor(mu) spans the whole grid for
    # every centre inside it; centres outside are shifted by the same rule.
    reach = 2 * max(w, h, c)
    half = (reach, reach, reach)
    params = D.cloud_to_params(cloud, dev)
    plan = D.FvrPlan(cloud.n, (w, h, c), half, 0, dev)
    vol = plan.new_volume()
    plan.bin(params)
    plan.forward(params, vol)
    return VolumeGrid.from_zyx(D.yxz_to_zyx(vol))


def backward(cloud: GaussianCloud, box: BoxConfig, dims, dl_dvol: VolumeGrid,
             prev: ParamGradients | None = None) -> ParamGradients:
    """Analytic adjoint of :func:`reconstruct` (fvr.py:227-273)."""
    w, h, c = _check_args(cloud, box, dims)
    if tuple(dl_dvol.dims) != (w, h, c):
        raise ValidationError(f"upstream gradient dims {dl_dvol.dims} != volume dims {(w, h, c)}")
    n = cloud.n
    if prev is not None and prev.d_mu.shape[0] != n:
        raise ValidationError(f"carried gradient stats have N = {prev.d_mu.shape[0]}, "
                              f"cloud has {n}")
    dev = D.require_cuda()
    params = D.cloud_to_params(cloud, dev)
    up = D.zyx_to_yxz(dl_dvol.zyx, dev)
    plan = D.FvrPlan(n, (w, h, c), box.half, 0, dev)
    plan.bin(params)
    grads = torch.empty((5, n), dtype=torch.float64, device=dev)
    accum = torch.zeros(n, dtype=torch.float64, device=dev)
    if prev is not None:
        accum.copy_(torch.from_numpy(np.asarray(prev.accum_pos_grad_norm)))
    plan.backward(params, up, grads, accum)
    g = grads.cpu().numpy()
    iters = 1 if prev is None else prev.iters_since_densify + 1
    return ParamGradients(np.ascontiguousarray(g[0:3].T), g[3], g[4], accum.cpu().numpy(), iters)
