"""CPU oracle of the cone-beam extension -- TEST INFRASTRUCTURE ONLY.

PARITY UNPINNED: the reference has no cone-beam geometry (SPEC.md:15,249,255
exclude it).  This module restates the model documented in
DESIGN.md "Cone beam" / csrc/cone.cu in plain Python + numpy (f64) so the CUDA
kernels can be checked on small cases.  The xy part is the reference's fan ray
(_kernels.py:208-259: _clip_ray, _ray_geometry; samples at t0 + (k + 1/2) step,
n_steps = int((t1 - t0) / step)) with its bilinear weights merged per pixel
(as the per-slice operator does); each (column, pixel) entry carries the
weight-averaged sample distance tbar, and detector row v reads the pixel's
z-column at z = cz + v tbar / L (L = |P - S|) by linear interpolation, zero
outside the volume, scaled by step * sqrt(1 + (v / L)^2).  It is pinned
indirectly by the tests: the centre row of an odd-c volume equals the
reference-pinned fan projection of slice cz, the adjoint passes the dot test,
and a ball's chord lengths match.
Only tests/ import it.
"""
from __future__ import annotations

import math

import numpy as np


def _clip_ray(px, py, dx, dy, t0, t1, xlo, xhi, ylo, yhi):
    # _kernels.py:208-229
    if dx != 0.0:
        ta, tb = (xlo - px) / dx, (xhi - px) / dx
        if ta > tb:
            ta, tb = tb, ta
        t0, t1 = max(t0, ta), min(t1, tb)
    elif px < xlo or px > xhi:
        return 1.0, 0.0
    if dy != 0.0:
        ta, tb = (ylo - py) / dy, (yhi - py) / dy
        if ta > tb:
            ta, tb = tb, ta
        t0, t1 = max(t0, ta), min(t1, tb)
    elif py < ylo or py > yhi:
        return 1.0, 0.0
    return t0, t1


def column_samples(cos_a, sin_a, u, rs, rd, w, h, step):
    """Fan ray of detector column u (_kernels.py:232-259) -> samples (x, y, tau), L."""
    cx, cy = 0.5 * (w - 1), 0.5 * (h - 1)
    sx, sy = cx - rs * cos_a, cy - rs * sin_a
    px, py = cx + rd * cos_a - u * sin_a, cy + rd * sin_a + u * cos_a
    dx, dy = px - sx, py - sy
    length = math.sqrt(dx * dx + dy * dy)
    dx, dy = dx / length, dy / length
    t0, t1 = _clip_ray(sx, sy, dx, dy, 0.0, length, -1.0, float(w), -1.0, float(h))
    out = []
    if t1 > t0:
        for k in range(int((t1 - t0) / step)):
            t = t0 + (k + 0.5) * step
            out.append((sx + t * dx, sy + t * dy, t / length))
    return out, length


def column_entries(samples, w, h):
    """Merge the bilinear taps of a column's samples (x, y, tau) per pixel ->
    {(x, y): (W, W tau)} (march_ray's merge, _kernels.py:279-300 taps)."""
    ent = {}
    for x, y, tau in samples:
        x0, y0 = math.floor(x), math.floor(y)
        fx, fy = x - x0, y - y0
        for xi, yi, wq in ((x0, y0, (1 - fx) * (1 - fy)), (x0 + 1, y0, fx * (1 - fy)),
                           (x0, y0 + 1, (1 - fx) * fy), (x0 + 1, y0 + 1, fx * fy)):
            if 0 <= xi < w and 0 <= yi < h and wq != 0.0:
                a, b = ent.get((xi, yi), (0.0, 0.0))
                ent[(xi, yi)] = (a + wq, b + wq * tau)
    return ent


def _lerp(col, z):
    z0 = math.floor(z)
    fz = z - z0
    acc = 0.0
    if 0 <= z0 < col.shape[0]:
        acc += (1 - fz) * col[z0]
    if 0 <= z0 + 1 < col.shape[0]:
        acc += fz * col[z0 + 1]
    return acc


def cone_forward(vol_zyx, geom, step=0.5, z0=0, c_global=None):
    """vol slab (c_local, h, w) -> partial cone projections (m, nu, nv), f64."""
    vol = np.asarray(vol_zyx, np.float64)
    cl, h, w = vol.shape
    cg = cl if c_global is None else int(c_global)
    zc = 0.5 * (cg - 1) - z0
    m, nu, nv = geom.n_views, geom.n_detectors, geom.n_rows
    sv, su = float(geom.row_spacing), float(geom.detector_spacing)
    rs, rd = float(geom.source_to_origin), float(geom.origin_to_detector)
    out = np.zeros((m, nu, nv))
    for a, ang in enumerate(np.asarray(geom.view_angles, np.float64)):
        ca, sa = math.cos(ang), math.sin(ang)
        for d in range(nu):
            u = (d - 0.5 * (nu - 1)) * su
            samples, length = column_samples(ca, sa, u, rs, rd, w, h, step)
            ent = column_entries(samples, w, h)
            for dv in range(nv):
                v = (dv - 0.5 * (nv - 1)) * sv
                acc = sum(W * _lerp(vol[:, yi, xi], zc + v * (WT / W))
                          for (xi, yi), (W, WT) in ent.items())
                out[a, d, dv] = acc * step * math.sqrt(1.0 + (v / length) ** 2)
    return out


def cone_forward_per_sample(vol_zyx, geom, step=0.5):
    """The same fan-ray samples, but every sample interpolates z at its OWN
    distance tau = t / L (trilinear per sample, no per-pixel merge): the
    finer model the merged one approximates.  Used to bound the merge error
    at large cone angles (tests/test_gpu_cone.py)."""
    vol = np.asarray(vol_zyx, np.float64)
    c, h, w = vol.shape
    zc = 0.5 * (c - 1)
    m, nu, nv = geom.n_views, geom.n_detectors, geom.n_rows
    sv, su = float(geom.row_spacing), float(geom.detector_spacing)
    rs, rd = float(geom.source_to_origin), float(geom.origin_to_detector)
    out = np.zeros((m, nu, nv))
    vs = (np.arange(nv) - 0.5 * (nv - 1)) * sv
    for a, ang in enumerate(np.asarray(geom.view_angles, np.float64)):
        ca, sa = math.cos(ang), math.sin(ang)
        for d in range(nu):
            u = (d - 0.5 * (nu - 1)) * su
            smp, length = column_samples(ca, sa, u, rs, rd, w, h, step)
            if not smp:
                continue
            smp = np.array(smp)
            x, y, tau = smp[:, 0], smp[:, 1], smp[:, 2]
            x0, y0 = np.floor(x).astype(int), np.floor(y).astype(int)
            fx, fy = x - x0, y - y0
            z = zc + tau[:, None] * vs[None, :]
            z0 = np.floor(z).astype(int)
            fz = z - z0
            acc = np.zeros(nv)
            for xi, yi, wq in ((x0, y0, (1 - fx) * (1 - fy)), (x0 + 1, y0, fx * (1 - fy)),
                               (x0, y0 + 1, (1 - fx) * fy), (x0 + 1, y0 + 1, fx * fy)):
                ok = (xi >= 0) & (xi < w) & (yi >= 0) & (yi < h)
                xc, yc = np.clip(xi, 0, w - 1)[:, None], np.clip(yi, 0, h - 1)[:, None]
                for zz, wz in ((z0, 1 - fz), (z0 + 1, fz)):
                    okz = ok[:, None] & (zz >= 0) & (zz < c)
                    val = np.where(okz, vol[np.clip(zz, 0, c - 1), yc, xc], 0.0)
                    acc += (wq[:, None] * wz * val).sum(0)
            out[a, d, :] = acc * step * np.sqrt(1.0 + (vs / length) ** 2)
    return out
