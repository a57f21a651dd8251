"""Synthetic phantoms (host-side input generation).

``shepp_logan_2d`` / ``shepp_logan_3d`` reproduce the reference's modified
Shepp-Logan rasterisation (phantom.py:1-94: same ellipse tables, grid
mapping to [-1, 1] with samples on the endpoints, additive values).
``chest_3d`` is new: a deterministic ellipsoid chest phantom
for the 256^3 configurations, values in [0, 1].
"""

from __future__ import annotations

import numpy as np

from .core import ValidationError, VolumeGrid

__all__ = ["chest_3d", "shepp_logan_2d", "shepp_logan_3d"]

# (value, semi-axis a, semi-axis b, centre x, centre y, rotation in degrees)
_SL2 = np.array([
    (1.0, 0.69, 0.92, 0.0, 0.0, 0.0),
    (-0.8, 0.6624, 0.874, 0.0, -0.0184, 0.0),
    (-0.2, 0.11, 0.31, 0.22, 0.0, -18.0),
    (-0.2, 0.16, 0.41, -0.22, 0.0, 18.0),
    (0.1, 0.21, 0.25, 0.0, 0.35, 0.0),
    (0.1, 0.046, 0.046, 0.0, 0.1, 0.0),
    (0.1, 0.046, 0.046, 0.0, -0.1, 0.0),
    (0.1, 0.046, 0.023, -0.08, -0.605, 0.0),
    (0.1, 0.023, 0.023, 0.0, -0.605, 0.0),
    (0.1, 0.023, 0.046, 0.06, -0.605, 0.0),
])

# (value, a, b, c, x0, y0, z0, rotation about z in degrees)
_SL3 = np.array([
    (1.0, 0.69, 0.92, 0.81, 0.0, 0.0, 0.0, 0.0),
    (-0.8, 0.6624, 0.874, 0.78, 0.0, -0.0184, 0.0, 0.0),
    (-0.2, 0.11, 0.31, 0.22, 0.22, 0.0, 0.0, -18.0),
    (-0.2, 0.16, 0.41, 0.28, -0.22, 0.0, 0.0, 18.0),
    (0.1, 0.21, 0.25, 0.41, 0.0, 0.35, -0.15, 0.0),
    (0.1, 0.046, 0.046, 0.05, 0.0, 0.1, 0.25, 0.0),
    (0.1, 0.046, 0.046, 0.05, 0.0, -0.1, 0.25, 0.0),
    (0.1, 0.046, 0.023, 0.05, -0.08, -0.605, 0.0, 0.0),
    (0.1, 0.023, 0.023, 0.02, 0.0, -0.605, 0.0, 0.0),
    (0.1, 0.023, 0.046, 0.05, 0.06, -0.605, 0.0, 0.0),
])

# chest: body, two lungs (air), heart, spine, aorta, sternum, ribs, nodules
_CHEST = [
    (0.60, 0.85, 0.62, 0.98, 0.0, 0.0, 0.0, 0.0),       # soft-tissue body
    (-0.52, 0.33, 0.44, 0.80, -0.38, 0.02, 0.05, 8.0),  # right lung
    (-0.52, 0.31, 0.42, 0.78, 0.38, 0.02, 0.05, -8.0),  # left lung
    (0.08, 0.22, 0.18, 0.35, 0.08, 0.10, -0.15, 25.0),  # heart
    (0.35, 0.09, 0.09, 0.98, 0.0, -0.47, 0.0, 0.0),     # vertebral column
    (0.05, 0.06, 0.06, 0.90, -0.05, -0.30, 0.0, 0.0),   # aorta
    (0.30, 0.10, 0.03, 0.60, 0.0, 0.56, 0.0, 0.0),      # sternum
    (0.20, 0.80, 0.58, 0.04, 0.0, 0.0, -0.55, 0.0),     # rib band (low)
    (0.20, 0.81, 0.59, 0.04, 0.0, 0.0, -0.15, 0.0),     # rib band
    (0.20, 0.82, 0.60, 0.04, 0.0, 0.0, 0.25, 0.0),      # rib band
    (0.20, 0.80, 0.58, 0.04, 0.0, 0.0, 0.65, 0.0),      # rib band (high)
    (0.45, 0.035, 0.035, 0.035, -0.42, 0.10, 0.20, 0.0),  # nodule
    (0.45, 0.025, 0.025, 0.025, 0.35, -0.12, -0.30, 0.0),  # nodule
]


def _axis(n: int) -> np.ndarray:
    return np.zeros(1) if n == 1 else np.linspace(-1.0, 1.0, n)


def _check(dims, min_side=32):
    for d in dims:
        if int(d) != 1 and int(d) < min_side:
            raise ValidationError(f"phantom axes must be >= {min_side} voxels (or 1), "
                                  f"got {tuple(dims)}")


def _rot(X, Y, x0, y0, deg):
    t = np.deg2rad(deg)
    ct, st = np.cos(t), np.sin(t)
    return (X - x0) * ct + (Y - y0) * st, -(X - x0) * st + (Y - y0) * ct


def shepp_logan_2d(w: int, h: int) -> VolumeGrid:
    """Single-slice head phantom on a (w, h, 1) grid (phantom.py:61-74)."""
    _check((w, h))
    X, Y = np.meshgrid(_axis(w), _axis(h), indexing="xy")
    img = np.zeros((h, w))
    for val, a, b, x0, y0, phi in _SL2:
        u, v = _rot(X, Y, x0, y0, phi)
        img[(u / a) ** 2 + (v / b) ** 2 <= 1.0] += val
    return VolumeGrid.from_zyx(img[None])


def _ellipsoids(table, w, h, c) -> np.ndarray:
    X, Y = np.meshgrid(_axis(w), _axis(h), indexing="xy")
    zs = _axis(c)
    vol = np.zeros((c, h, w))
    for val, a, b, cc, x0, y0, z0, phi in table:
        u, v = _rot(X, Y, x0, y0, phi)
        q = (u / a) ** 2 + (v / b) ** 2
        for k, z in enumerate(zs):
            dz = ((z - z0) / cc) ** 2
            if dz <= 1.0:
                vol[k][q <= 1.0 - dz] += val
    return vol


def shepp_logan_3d(w: int, h: int, c: int) -> VolumeGrid:
    """Volumetric head phantom (phantom.py:76-94)."""
    _check((w, h, c))
    return VolumeGrid.from_zyx(_ellipsoids(_SL3, w, h, c))


def chest_3d(w: int, h: int, c: int) -> VolumeGrid:
    """Deterministic ellipsoid chest phantom, values clipped to [0, 1]."""
    _check((w, h, c))
    return VolumeGrid.from_zyx(np.clip(_ellipsoids(_CHEST, w, h, c), 0.0, 1.0))
