"""CPU oracle for the DGR hot path -- TEST INFRASTRUCTURE ONLY.

A restatement of the reference's algorithm (``/root/reference/pkg/src/splatct``)
on plain numpy arrays, with the heavy loops in ``oracle.c`` (double precision,
OpenMP).  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU
baseline legs may import this module, and only as the checker / the timed
CPU baseline.  The product package never imports it.

Parity of this restatement is pinned against golden vectors produced by the
reference itself (``tests/golden/make_golden.py`` -> ``tests/golden/*.npz``;
checked by ``tests/test_oracle_golden.py``).

Every function cites the reference code it restates.  Stage-boundary float32
quantisation follows the reference loop (optim.py:350-403): volumes, sinograms
and the volume gradient are stored as float32 between stages
(core.py:69,109; optim.py:368,371).
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i32p = ctypes.POINTER(ctypes.c_int32)
_i64p = ctypes.POINTER(ctypes.c_int64)


def build() -> str:
    """Compile oracle.c (gcc -fopenmp) into oracle/_build/liboracle.so."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH) or (
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "oracle.c"))
        ):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        i64, i32, d = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        L.or_splat_fwd.argtypes = [_dp, _dp, _dp, i64, i32, i32, i32, i32, i32, i32, _dp]
        L.or_splat_plain.argtypes = L.or_splat_fwd.argtypes
        L.or_splat_bwd.argtypes = [_dp, _dp, _dp, i64, i32, i32, i32, i32, i32, i32, _dp,
                                   _dp, _dp, _dp]
        L.or_bins.argtypes = [_dp, i64, i32, i32, i32, i32, i32, i32, i32, i32, i32, _i32p,
                              _i64p, _i32p]
        L.or_bins.restype = i64
        L.or_project_forward.argtypes = [_dp, _dp, _dp, _dp, i32, i32, i32, i32, i32, d, d,
                                         i32, d, d]
        L.or_project_adjoint.argtypes = L.or_project_forward.argtypes
        L.or_ssim_slices.argtypes = [_dp, _dp, i32, i32, i32, _dp, i32, _dp, i32, d, d, _dp,
                                     _dp]
        L.or_num_threads.restype = i32
        L.or_set_num_threads.argtypes = [i32]
        _lib = L
    return _lib


def num_threads() -> int:
    return int(lib().or_num_threads())


def set_num_threads(n: int) -> None:
    lib().or_set_num_threads(int(n))


def _p(a, t=_dp):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# --------------------------------------------------------------------------
# voxelizer (fvr.py:148-273, _kernels.py:22-205)
# --------------------------------------------------------------------------

def box_half(box):
    """BoxConfig.half (core.py:166-168) for a (w0, h0, c0) odd box."""
    return tuple((int(b) - 1) // 2 for b in box)


def splat_fwd(mu, sigma, intensity, box, dims) -> np.ndarray:
    """fvr.reconstruct (fvr.py:148-167) -> float32 (c,h,w) like VolumeGrid."""
    mu, sigma, intensity = _f64(mu), _f64(sigma), _f64(intensity)
    w, h, c = (int(v) for v in dims)
    hx, hy, hz = box_half(box)
    vol = np.zeros((c, h, w), np.float64)
    lib().or_splat_fwd(_p(mu), _p(sigma), _p(intensity), mu.shape[0], hx, hy, hz, w, h, c,
                       _p(vol))
    return vol.astype(np.float32)


def splat_plain(mu, sigma, intensity, box, dims) -> np.ndarray:
    """fvr.reconstruct_nodecomp (fvr.py:170-190)."""
    mu, sigma, intensity = _f64(mu), _f64(sigma), _f64(intensity)
    w, h, c = (int(v) for v in dims)
    hx, hy, hz = box_half(box)
    vol = np.zeros((c, h, w), np.float64)
    lib().or_splat_plain(_p(mu), _p(sigma), _p(intensity), mu.shape[0], hx, hy, hz, w, h,
                         c, _p(vol))
    return vol.astype(np.float32)


def splat_direct(mu, sigma, intensity, dims) -> np.ndarray:
    """fvr.reconstruct_direct (fvr.py:193-224): unconfined dense sum."""
    w, h, c = (int(v) for v in dims)
    xs, ys, zs = (np.arange(k, dtype=np.float64) for k in (w, h, c))
    out = np.zeros((c, h, w))
    for i in range(len(sigma)):
        mx, my, mz = mu[i]
        inv2 = 0.5 / sigma[i] ** 2
        d2 = ((zs - mz) ** 2)[:, None, None] + ((ys - my) ** 2)[None, :, None] + \
            ((xs - mx) ** 2)[None, None, :]
        out += intensity[i] * np.exp(-inv2 * d2)
    return out.astype(np.float32)


def splat_bwd(mu, sigma, intensity, box, dims, upstream, prev_accum=None, prev_iters=0):
    """fvr.backward (fvr.py:227-273). upstream: float32 (c,h,w).

    Returns (d_mu (N,3), d_sigma, d_intensity, accum_pos_grad_norm, iters).
    """
    mu, sigma, intensity = _f64(mu), _f64(sigma), _f64(intensity)
    w, h, c = (int(v) for v in dims)
    hx, hy, hz = box_half(box)
    n = mu.shape[0]
    up = _f64(np.asarray(upstream, dtype=np.float32))
    d_mu = np.zeros((n, 3))
    d_sigma = np.zeros(n)
    d_int = np.zeros(n)
    lib().or_splat_bwd(_p(mu), _p(sigma), _p(intensity), n, hx, hy, hz, w, h, c, _p(up),
                       _p(d_mu), _p(d_sigma), _p(d_int))
    pos = np.sqrt((d_mu * d_mu).sum(axis=1))
    if prev_accum is None:
        return d_mu, d_sigma, d_int, pos, 1
    return d_mu, d_sigma, d_int, prev_accum + pos, prev_iters + 1


def bins(mu, box, dims, tile):
    """Footprints + tile bin lists (CPU restatement).

    Returns (fp (N,6) int32 [xlo,xhi,ylo,yhi,zlo,zhi], tile_start (T+1,) int64,
    items (P,) int32 Gaussian ids, per tile in ascending id order).
    """
    mu = _f64(mu)
    w, h, c = (int(v) for v in dims)
    hx, hy, hz = box_half(box)
    tx, ty, tz = (int(t) for t in tile)
    n = mu.shape[0]
    nt = (-(-w // tx)) * (-(-h // ty)) * (-(-c // tz))
    fp = np.zeros((n, 6), np.int32)
    ts = np.zeros(nt + 1, np.int64)
    npairs = lib().or_bins(_p(mu), n, hx, hy, hz, w, h, c, tx, ty, tz, _p(fp, _i32p),
                           _p(ts, _i64p), ctypes.cast(None, _i32p))
    items = np.zeros(max(npairs, 1), np.int32)
    lib().or_bins(_p(mu), n, hx, hy, hz, w, h, c, tx, ty, tz, _p(fp, _i32p), _p(ts, _i64p),
                  _p(items, _i32p))
    return fp, ts, items[:npairs]


# --------------------------------------------------------------------------
# projector (projector.py:59-111, _kernels.py:208-357)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Geometry:
    """The per-slice geometry fields _geom_params reads (projector.py:50-56)."""

    is_fan: bool
    angles: np.ndarray
    n_det: int
    spacing: float
    rs: float = 0.0
    rd: float = 0.0

    @classmethod
    def parallel(cls, m, n, spacing=1.0, start=0.0, extent=np.pi):
        """ScanGeometry.parallel (core.py:353-359)."""
        return cls(False, start + extent * np.arange(m) / m, n, float(spacing))

    @classmethod
    def fan(cls, m, n, spacing, rs, rd, start=0.0, extent=np.pi):
        """ScanGeometry.fan (core.py:361-371)."""
        return cls(True, start + extent * np.arange(m) / m, n, float(spacing), float(rs),
                   float(rd))

    @property
    def m(self):
        return len(self.angles)


def project_forward(vol, geom: Geometry, step=0.5) -> np.ndarray:
    """forward_project (projector.py:59-77): vol (c,h,w) -> float32 (m,n,p)."""
    v = _f64(np.asarray(vol, dtype=np.float32))
    c, h, w = v.shape
    cos_t, sin_t = _f64(np.cos(geom.angles)), _f64(np.sin(geom.angles))
    sino = np.zeros((geom.m, geom.n_det, c))
    lib().or_project_forward(_p(v), _p(sino), _p(cos_t), _p(sin_t), geom.m, geom.n_det, c,
                             w, h, geom.spacing, float(step), int(geom.is_fan), geom.rs,
                             geom.rd)
    return sino.astype(np.float32)


def project_adjoint(sino, geom: Geometry, dims, step=0.5) -> np.ndarray:
    """back_project (projector.py:80-111): sino (m,n,p) -> float32 (c,h,w)."""
    s = _f64(np.asarray(sino, dtype=np.float32))
    w, h, c = (int(v) for v in dims)
    cos_t, sin_t = _f64(np.cos(geom.angles)), _f64(np.sin(geom.angles))
    vol = np.zeros((c, h, w))
    lib().or_project_adjoint(_p(s), _p(vol), _p(cos_t), _p(sin_t), geom.m, geom.n_det, c, w,
                             h, geom.spacing, float(step), int(geom.is_fan), geom.rs, geom.rd)
    return vol.astype(np.float32)


# --------------------------------------------------------------------------
# loss (loss.py:35-253)
# --------------------------------------------------------------------------

def gaussian_window(k: int, sigma: float = 1.5) -> np.ndarray:
    """_gaussian_window (loss.py:77-80)."""
    x = np.arange(k, dtype=np.float64) - (k - 1) / 2.0
    g = np.exp(-0.5 * (x / sigma) ** 2)
    return g / g.sum()


def ssim_windows(shape):
    """_ssim_windows (loss.py:104-109)."""
    kr = min(11, shape[0])
    kc = min(11, shape[1])
    kr -= 1 - kr % 2
    kc -= 1 - kc % 2
    return gaussian_window(kr), gaussian_window(kc)


def l1_loss(pred, ref):
    """l1_loss (loss.py:64-74)."""
    diff = np.asarray(pred, np.float32).astype(np.float64) - np.asarray(ref, np.float32)
    return float(np.abs(diff).sum() / diff.size), np.sign(diff) / diff.size


def ssim_stats_constants(ref):
    """L = max(ref) (<=0 -> 1), C1, C2 (loss.py:168-172)."""
    lmax = float(np.asarray(ref, np.float64).max())
    if lmax <= 0:
        lmax = 1.0
    return lmax, (0.01 * lmax) ** 2, (0.03 * lmax) ** 2


def ssim_loss(pred, ref, want_grad=True):
    """ssim_loss (loss.py:159-180) -> (1 - mean SSIM, grad (m,n,p))."""
    x = _f64(np.asarray(pred, np.float32))
    y = _f64(np.asarray(ref, np.float32))
    m, n, p = x.shape
    _, c1, c2 = ssim_stats_constants(y)
    gr, gc = ssim_windows((m, n))
    per = np.zeros(p)
    grad = np.zeros((m, n, p)) if want_grad else None
    lib().or_ssim_slices(_p(x), _p(y), m, n, p, _p(gr), len(gr), _p(gc), len(gc), c1, c2,
                         _p(per), _p(grad) if want_grad else ctypes.cast(None, _dp))
    mean = float(per.sum() / p)
    return 1.0 - mean, (-grad / p if want_grad else None)


def ssim_value(x, y, max_val=None) -> float:
    """ssim_value (loss.py:144-156) for one 2D image pair."""
    x = _f64(x)[:, :, None]
    y = _f64(y)[:, :, None]
    lmax = float(np.max(y)) if max_val is None else float(max_val)
    if lmax <= 0:
        lmax = 1.0
    c1, c2 = (0.01 * lmax) ** 2, (0.03 * lmax) ** 2
    gr, gc = ssim_windows(x.shape[:2])
    per = np.zeros(1)
    lib().or_ssim_slices(_p(x), _p(y), x.shape[0], x.shape[1], 1, _p(gr), len(gr), _p(gc),
                         len(gc), c1, c2, _p(per), ctypes.cast(None, _dp))
    return float(per[0])


def tv_loss(vol):
    """tv_loss (loss.py:183-207): vol (c,h,w) -> (value, grad (c,h,w))."""
    v = np.asarray(vol, np.float32).astype(np.float64)
    count = v.size
    total = 0.0
    grad = np.zeros_like(v)
    for axis in range(3):
        if v.shape[axis] < 2:
            continue
        d = np.diff(v, axis=axis)
        total += np.abs(d).sum()
        s = np.sign(d)
        lead = [slice(None)] * 3
        lag = [slice(None)] * 3
        lead[axis] = slice(1, None)
        lag[axis] = slice(0, -1)
        grad[tuple(lead)] += s
        grad[tuple(lag)] -= s
    return total / count, grad / count


def total_loss_detailed(pred, ref, vol, lambdas=(0.6, 0.2, 1.0)):
    """total_loss_detailed (loss.py:210-239)."""
    l1w, ssw, tvw = lambdas
    value = 0.0
    parts = {"l1": float("nan"), "ssim": float("nan"), "tv": float("nan")}
    gp = np.zeros(np.shape(pred))
    gv = np.zeros(np.shape(vol))
    if l1w > 0:
        v, g = l1_loss(pred, ref)
        parts["l1"] = v
        value += l1w * v
        gp += l1w * g
    if ssw > 0:
        v, g = ssim_loss(pred, ref)
        parts["ssim"] = v
        value += ssw * v
        gp += ssw * g
    if tvw > 0:
        v, g = tv_loss(vol)
        parts["tv"] = v
        value += tvw * v
        gv += tvw * g
    return value, gp, gv, parts


# --------------------------------------------------------------------------
# optimizer + loop (optim.py:61-144, 286-427)
# --------------------------------------------------------------------------

ADAM_BETA1, ADAM_BETA2, ADAM_EPS, SIGMA_FLOOR = 0.9, 0.999, 1e-8, 0.3


def lr_at(step, lr0, lrf, max_iters):
    """OptimizerState.lr (optim.py:88-90), pre-increment step."""
    t = min(step, max_iters) / max(max_iters, 1)
    return lr0 * (lrf / lr0) ** t


def adam_step(mu, sigma, inten, d_mu, d_sigma, d_int, st, sigma_ceiling):
    """adam_step (optim.py:109-144).  st: dict with m_*/v_* arrays, step, lr0,
    lrf, max_iters.  Returns (mu, sigma, inten, new_state)."""
    t = st["step"] + 1
    lr = lr_at(st["step"], st["lr0"], st["lrf"], st["max_iters"])
    bc1 = 1.0 - ADAM_BETA1 ** t
    bc2 = 1.0 - ADAM_BETA2 ** t

    def upd(p, g, m, v):
        m = ADAM_BETA1 * m + (1 - ADAM_BETA1) * g
        v = ADAM_BETA2 * v + (1 - ADAM_BETA2) * g * g
        return p - lr * (m / bc1) / (np.sqrt(v / bc2) + ADAM_EPS), m, v

    mu, m_mu, v_mu = upd(mu, d_mu, st["m_mu"], st["v_mu"])
    sigma, m_s, v_s = upd(sigma, d_sigma, st["m_sigma"], st["v_sigma"])
    inten, m_i, v_i = upd(inten, d_int, st["m_intensity"], st["v_intensity"])
    sigma = np.clip(sigma, SIGMA_FLOOR, sigma_ceiling)
    inten = np.maximum(inten, 0.0)
    ns = dict(st, m_mu=m_mu, v_mu=v_mu, m_sigma=m_s, v_sigma=v_s, m_intensity=m_i,
              v_intensity=v_i, step=t)
    return mu, sigma, inten, ns


def fresh_state(n, lr0=3e-4, lrf=3e-5, max_iters=1000):
    z = np.zeros
    return dict(m_mu=z((n, 3)), v_mu=z((n, 3)), m_sigma=z(n), v_sigma=z(n),
                m_intensity=z(n), v_intensity=z(n), step=0, lr0=lr0, lrf=lrf,
                max_iters=max_iters)


def psnr(x, y, max_val=None):
    """metrics.psnr (metrics.py:24-38)."""
    x = np.asarray(x, np.float64)
    y = np.asarray(y, np.float64)
    peak = float(np.max(y)) if max_val is None else float(max_val)
    mse = float(np.mean((x - y) ** 2))
    if mse == 0.0:
        return 200.0
    return min(10.0 * np.log10(peak * peak / mse), 200.0)


def train(meas, geom: Geometry, dims, box, mu, sigma, inten, max_iters, lambdas=(0.6, 0.2, 1.0),
          lr0=3e-4, lrf=3e-5, iters_to_run=None, truth=None, step=0.5):
    """run_reconstruction loop body (optim.py:350-415), densify off
    (densify_interval=0), stop_rule "iters", given init cloud.

    Returns (volume f32 (c,h,w), (mu, sigma, inten), trace list of dicts).
    """
    mu, sigma, inten = _f64(mu).copy(), _f64(sigma).copy(), _f64(inten).copy()
    st = fresh_state(len(sigma), lr0, lrf, max_iters)
    sigma_ceiling = 3.0 * max(box)
    run = max_iters if iters_to_run is None else min(iters_to_run, max_iters)
    vol = splat_fwd(mu, sigma, inten, box, dims)
    accum, iters_acc = None, 0
    trace = []
    for it in range(run):
        pred = project_forward(vol, geom, step)
        value, gp, gv, parts = total_loss_detailed(pred, meas, vol, lambdas)
        if not np.isfinite(value):
            raise FloatingPointError(f"non-finite loss at iteration {it}")
        data_grad = project_adjoint(gp.astype(np.float32), geom, dims, step).astype(np.float64)
        dl = (data_grad + gv).astype(np.float32)
        d_mu, d_s, d_i, accum, iters_acc = splat_bwd(mu, sigma, inten, box, dims, dl, accum,
                                                     iters_acc)
        mu, sigma, inten, st = adam_step(mu, sigma, inten, d_mu, d_s, d_i, st, sigma_ceiling)
        vol = splat_fwd(mu, sigma, inten, box, dims)
        row = dict(iteration=it + 1, loss=value, l1=parts["l1"], ssim=parts["ssim"],
                   tv=parts["tv"])
        if truth is not None:
            row["psnr"] = psnr(vol, truth)
        trace.append(row)
    return vol, (mu, sigma, inten), trace
