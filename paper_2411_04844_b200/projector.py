"""Geometry transform between volume and projection domains (B200).

Drop-in for the reference's ``splatct.projector`` (projector.py:1-239).
``forward_project`` / ``back_project`` apply the exact sampled operator A /
A^T built once per geometry on the device (device.ProjectorOperator; the
reference's Joseph-style sampling, _kernels.py:208-357).  ``fbp`` runs its
ramp filter and pixel-driven back projection on the device (csrc/fbp.cu);
the 1D filter kernel itself is tabulated on the host exactly as
``_ramp_response`` defines it.  ``add_noise`` is host-side data simulation
(numpy RNG, bit-identical to the reference for a given seed).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import device as D
from ._lib import call
from .core import ScanGeometry, Sinogram, ValidationError, VolumeGrid

__all__ = ["RaySamplingConfig", "add_noise", "back_project", "cone_init_volume", "fbp",
           "forward_project"]


@dataclass(frozen=True)
class RaySamplingConfig:
    """Uniform bilinear sampling of the line integral (projector.py:37-47)."""

    step_length: float = 0.5

    def __post_init__(self):
        if not 0 < self.step_length <= 1:
            raise ValidationError(f"step_length must be in (0, 1], got {self.step_length}")


def forward_project(volume: VolumeGrid, geom: ScanGeometry,
                    sampling: RaySamplingConfig = RaySamplingConfig()) -> Sinogram:
    """Line integrals of every slice along every ray (projector.py:59-77)."""
    geom.check_volume(volume.dims)
    w, h, c = volume.dims
    dev = D.require_cuda()
    op = D.operator_for(geom, w, h, c, sampling.step_length, dev)
    vol = D.zyx_to_yxz(volume.zyx, dev)
    sino = op.forward(vol)
    return Sinogram.from_views(sino.cpu().numpy())


def back_project(sino: Sinogram, geom: ScanGeometry, dims,
                 sampling: RaySamplingConfig = RaySamplingConfig(),
                 deterministic: bool = False) -> VolumeGrid:
    """Exact adjoint of :func:`forward_project` (projector.py:80-111).

    Always deterministic on the device (CSR rows summed in a fixed order).
    """
    m, n, p = sino.dims
    w, h, c = (int(v) for v in dims)
    if (m, n) != (geom.n_views, geom.n_detectors):
        raise ValidationError(f"sinogram dims {sino.dims} do not match geometry "
                              f"({geom.n_views} views x {geom.n_detectors} detectors)")
    if p != geom.sino_depth(c):
        raise ValidationError(f"sinogram depth {p} does not match {geom.sino_depth(c)} "
                              f"({geom.variant} geometry, volume has {c} slices)")
    geom.check_volume(dims)
    dev = D.require_cuda()
    op = D.operator_for(geom, w, h, c, sampling.step_length, dev)
    g = D.sino_to_device(sino.views, dev)
    out = op.adjoint(g, c_local=c)
    return VolumeGrid.from_zyx(D.yxz_to_zyx(out))


def cone_init_volume(sino: Sinogram, geom: ScanGeometry, dims,
                     sampling: RaySamplingConfig = RaySamplingConfig()) -> VolumeGrid:
    """Initialiser volume for cone beam (the reference's FBP is per-slice only):
    the normalised back projection A^T y / A^T A 1, clipped at 0."""
    w, h, c = (int(v) for v in dims)
    dev = D.require_cuda()
    op = D.cone_projector_for(geom, w, h, c, sampling.step_length, dev)
    bp = op.adjoint(D.sino_to_device(sino.views, dev), c_local=c)
    norm = op.adjoint(op.forward(torch.ones((h, w, c), dtype=torch.float32, device=dev)),
                      c_local=c)
    vol = torch.where(norm > 1e-6 * norm.max(), bp / norm.clamp_min(1e-30),
                      torch.zeros_like(bp)).clamp_min(0)
    return VolumeGrid.from_zyx(D.yxz_to_zyx(vol))


def _ramp_response(n_pad: int, spacing: float, window: str) -> np.ndarray:
    """Band-limited ramp (Ram-Lak) frequency response (projector.py:114-131)."""
    k = np.arange(-(n_pad // 2), n_pad - n_pad // 2)
    imp = np.zeros(n_pad)
    imp[k == 0] = 1.0 / (4.0 * spacing ** 2)
    odd = (k % 2) != 0
    imp[odd] = -1.0 / (np.pi ** 2 * k[odd].astype(np.float64) ** 2 * spacing ** 2)
    resp = np.real(np.fft.fft(np.fft.ifftshift(imp)))
    if window == "hann":
        resp *= 0.5 * (1.0 + np.cos(2.0 * np.pi * np.fft.fftfreq(n_pad)))
    elif window != "ramp":
        raise ValidationError(f"unknown filter {window!r}; use 'ramp' or 'hann'")
    return resp


def _filter_kernel(n: int, spacing: float, window: str) -> np.ndarray:
    """Real-space taps of _filter_rows (projector.py:134-141) for lags -(n-1)..n-1.

    Zero-padded FFT filtering of a length-n row is the circular convolution
    with h = ifft(resp); no wrap-around reaches the first n outputs because
    n_pad >= 2n, so out[i] = spacing * sum_j h[(i-j) mod n_pad] x[j].
    """
    n_pad = int(2 ** np.ceil(np.log2(max(64, 2 * n))))
    h = np.real(np.fft.ifft(_ramp_response(n_pad, spacing, window)))
    lags = np.arange(-(n - 1), n)
    return np.ascontiguousarray(h[lags % n_pad] * spacing)


def _angular_weight(geom: ScanGeometry) -> float:
    """Per-view weight, halved on near-full-circle coverage (projector.py:144-151)."""
    a = geom.view_angles
    if geom.n_views < 2:
        return float(np.pi)
    dbeta = float(np.mean(np.diff(a)))
    span = float(a[-1] - a[0]) + dbeta
    return 0.5 * dbeta if span > 1.5 * np.pi else dbeta


def fbp_device(sino_dev: torch.Tensor, geom: ScanGeometry, dims,
               filter_name: str = "ramp") -> torch.Tensor:
    """FBP of a device sinogram (m, n, p) -> device volume (h, w, p)."""
    m, n, p = (int(v) for v in sino_dev.shape)
    w, h, c = (int(v) for v in dims)
    dev = sino_dev.device
    if geom.variant == "parallel":
        spacing = float(geom.detector_spacing)
        wdet = None
        rs = 0.0
    else:
        rs = float(geom.source_to_origin)
        rd = float(geom.origin_to_detector)
        spacing = float(geom.detector_spacing) * rs / (rs + rd)
        u_iso = (np.arange(n) - 0.5 * (n - 1)) * spacing
        wdet = torch.from_numpy(rs / np.sqrt(rs ** 2 + u_iso ** 2)).to(dev)
    kern = torch.from_numpy(_filter_kernel(n, spacing, filter_name)).to(dev)
    filt = torch.empty((m, n, p), dtype=torch.float64, device=dev)
    call("splatct_fbp_filter", D.ptr(sino_dev), m, n, p, D.ptr(kern), D.ptr(wdet), D.ptr(filt),
         D.stream_handle())
    ang = np.asarray(geom.view_angles, np.float64)
    cos_t = torch.from_numpy(np.cos(ang)).to(dev)
    sin_t = torch.from_numpy(np.sin(ang)).to(dev)
    out = torch.empty((h, w, p), dtype=torch.float32, device=dev)
    call("splatct_fbp_backproject", D.ptr(filt), D.ptr(cos_t), D.ptr(sin_t), m, n, p, w, h,
         spacing, _angular_weight(geom), int(geom.variant == "fan"), rs, D.ptr(out),
         D.stream_handle())
    return out


def fbp(sino: Sinogram, geom: ScanGeometry, dims, filter_name: str = "ramp") -> VolumeGrid:
    """Filtered back projection, per slice (projector.py:154-206)."""
    m, n, p = sino.dims
    if m < 2:
        raise ValidationError("FBP needs at least 2 views")
    w, h, c = (int(v) for v in dims)
    if not geom.per_slice:
        raise ValidationError("FBP is per-slice (parallel / fan); cone beam initialises with "
                              "cone_init_volume")
    if p != c:
        raise ValidationError(f"sinogram has {p} slices, volume has {c}")
    geom.check_volume(dims)
    if filter_name not in ("ramp", "hann"):
        raise ValidationError(f"unknown filter {filter_name!r}; use 'ramp' or 'hann'")
    dev = D.require_cuda()
    out = fbp_device(D.sino_to_device(sino.views, dev), geom, dims, filter_name)
    return VolumeGrid.from_zyx(D.yxz_to_zyx(out))


def add_noise(sino: Sinogram, model: str = "gaussian", sigma: float = 0.0,
              photon_count: float = 1e5, seed: int = 0) -> Sinogram:
    """Reproducible measurement noise (projector.py:209-239); host numpy RNG."""
    rng = np.random.default_rng(seed)
    vals = sino.views.astype(np.float64)
    if model == "gaussian":
        if sigma < 0:
            raise ValidationError(f"gaussian sigma must be >= 0, got {sigma}")
        if sigma == 0:
            return Sinogram(sino.dims, sino.data.copy())
        noisy = vals + sigma * rng.standard_normal(vals.shape)
    elif model == "poisson":
        if photon_count <= 0:
            raise ValidationError(f"photon_count must be positive, got {photon_count}")
        counts = rng.poisson(photon_count * np.exp(-vals)).astype(np.float64)
        noisy = -np.log(np.maximum(counts, 1.0) / photon_count)
    else:
        raise ValidationError(f"unknown noise model {model!r}")
    return Sinogram.from_views(noisy)
