"""Generate golden input/output vectors by running the REAL reference.

This script is the only place that imports the reference package
(``/root/reference/pkg/src/splatct``, numba + numpy + scipy).  It runs in the
build container (where ``/root/reference`` exists) and writes small
``.npz`` fixtures next to itself; those fixtures travel with the repo and
are what the CPU oracle tests and the GPU parity tests compare against.

Usage (from the repo root):

    NUMBA_CACHE_DIR=/tmp/numba_ref python tests/golden/make_golden.py [--traj]

``--traj`` additionally runs the config-1 500-iteration trajectory
(64^3 Shepp-Logan, 10k Gaussians, 25-view parallel beam; ~2 min on 8 cores)
and stores its init cloud, loss trace and final metrics.

Reference call sites exercised (file:line in /root/reference/pkg/src/splatct):
  fvr.reconstruct            fvr.py:148    (-> _kernels.splat_decomposed :22)
  fvr.backward               fvr.py:227    (-> _kernels.splat_backward   :132)
  projector.forward_project  projector.py:59 (-> _kernels.project_forward :262)
  projector.back_project     projector.py:80 (-> _kernels.project_adjoint :306)
  loss.l1_loss / ssim_loss / tv_loss / total_loss_detailed  loss.py:64-239
  optim.adam_step            optim.py:109
  optim.run_reconstruction   optim.py:286
  densify.densify_and_prune  densify.py:86  + OptimizerState.remap optim.py:92
                             (-> densify.npz; ``--only densify`` writes just that)
  headline pins (``--only c2pins`` -> c2pins.npz): SURVEY section 8(c)'s short
  C2/C3 runs -- 256^3 Shepp-Logan, fan(50|25, 512, 1.6, 512, 512), FBP init
  (projector.fbp :154 + optim.init_cloud_fbp :158, seed 0, 50k), 4 iterations
  of optim.run_reconstruction :286 with deterministic=True, densify off.
"""

from __future__ import annotations

import argparse
import os
import sys
import time

import numpy as np

REF_SRC = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_ref")
sys.path.insert(0, REF_SRC)

import splatct  # noqa: E402  (the reference)
from splatct import core, densify, fvr, loss, optim, phantom, projector, metrics  # noqa: E402

assert os.path.dirname(splatct.__file__).startswith(REF_SRC), splatct.__file__


def cloud_arrays(cl):
    return dict(mu=np.array(cl.mu), sigma=np.array(cl.sigma), intensity=np.array(cl.intensity))


def rand_cloud(rng, n, dims, margin=-3.0, smin=0.4, smax=2.5):
    """Params generated in float32 then widened (survey section 7.1)."""
    w, h, c = dims
    lo = np.array([margin, margin, margin])
    hi = np.array([w, h, c], dtype=float) - margin
    mu = rng.uniform(lo, hi, (n, 3)).astype(np.float32).astype(np.float64)
    sigma = rng.uniform(smin, smax, n).astype(np.float32).astype(np.float64)
    inten = rng.uniform(0.0, 1.0, n).astype(np.float32).astype(np.float64)
    return core.GaussianCloud(mu, sigma, inten)


def gen_fvr(out):
    rng = np.random.default_rng(1234)
    cases = [
        # (dims, box, n)
        ((32, 32, 32), (17, 17, 17), 60),
        ((40, 24, 12), (17, 9, 5), 80),     # non-cubic box, per-axis halves differ
        ((20, 20, 20), (17, 17, 17), 25),   # box nearly the whole volume
        ((33, 17, 19), (7, 7, 7), 150),     # odd dims, small box
    ]
    for ci, (dims, box, n) in enumerate(cases):
        cl = rand_cloud(rng, n, dims)
        # a few exact-integer and negative-floor centres
        mu = np.array(cl.mu)
        mu[0] = [8.0, 8.0, 8.0]
        mu[1] = [-0.5, 3.25, 2.0]          # floor(-0.5) = -1: true floor, not trunc
        mu[2] = [dims[0] - 0.25, dims[1] + 1.5, 1.0]  # outside in y
        cl = core.GaussianCloud(mu, cl.sigma, cl.intensity)
        bx = core.BoxConfig(*box)
        import warnings
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            vol = fvr.reconstruct(cl, bx, dims, deterministic=True)
            up = rng.standard_normal(dims[::-1]).astype(np.float32)
            up[0, 0, :3] = 0.0
            g = fvr.backward(cl, bx, dims, core.VolumeGrid.from_zyx(up))
        out[f"fvr{ci}_dims"] = np.array(dims)
        out[f"fvr{ci}_box"] = np.array(box)
        for k, v in cloud_arrays(cl).items():
            out[f"fvr{ci}_{k}"] = v
        out[f"fvr{ci}_vol"] = vol.zyx.copy()
        out[f"fvr{ci}_up"] = up
        out[f"fvr{ci}_d_mu"] = np.array(g.d_mu)
        out[f"fvr{ci}_d_sigma"] = np.array(g.d_sigma)
        out[f"fvr{ci}_d_intensity"] = np.array(g.d_intensity)
        out[f"fvr{ci}_accum"] = np.array(g.accum_pos_grad_norm)
    out["fvr_ncases"] = np.array(len(cases))
    # SPEC.md:134-135 known answers
    dims = (17, 17, 17)
    bx = core.BoxConfig.cube(17)
    v1 = fvr.reconstruct(core.GaussianCloud([[8, 8, 8]], [1.0], [1.0]), bx, dims)
    v2 = fvr.reconstruct(core.GaussianCloud([[8.5, 8, 8]], [1.0], [1.0]), bx, dims)
    out["spec_v_int"] = v1.zyx.copy()
    out["spec_v_half"] = v2.zyx.copy()


def gen_proj(out):
    rng = np.random.default_rng(99)
    cases = [
        ("parallel", (24, 20, 3), dict(n_views=7, n_detectors=30, detector_spacing=1.0)),
        ("parallel", (16, 16, 2), dict(n_views=5, n_detectors=23, detector_spacing=0.7,
                                       angle_start=0.1, angle_extent=2.0)),
        ("fan", (24, 20, 3), dict(n_views=9, n_detectors=40, detector_spacing=1.3,
                                  source_to_origin=40.0, origin_to_detector=30.0)),
        ("fan", (13, 21, 2), dict(n_views=6, n_detectors=17, detector_spacing=2.1,
                                  source_to_origin=25.0, origin_to_detector=15.0,
                                  angle_start=0.3, angle_extent=5.5)),
    ]
    for ci, (variant, dims, kw) in enumerate(cases):
        if variant == "parallel":
            geom = core.ScanGeometry.parallel(**kw)
        else:
            geom = core.ScanGeometry.fan(**kw)
        w, h, c = dims
        vol = rng.uniform(0, 1, (c, h, w)).astype(np.float32)
        sino = projector.forward_project(core.VolumeGrid.from_zyx(vol), geom)
        ys = rng.standard_normal((geom.n_views, geom.n_detectors, c)).astype(np.float32)
        ys[0, :2, :] = 0.0
        bp = projector.back_project(core.Sinogram.from_views(ys), geom, dims, deterministic=True)
        out[f"proj{ci}_variant"] = np.array(variant)
        out[f"proj{ci}_dims"] = np.array(dims)
        out[f"proj{ci}_angles"] = np.array(geom.view_angles)
        out[f"proj{ci}_n_det"] = np.array(geom.n_detectors)
        out[f"proj{ci}_spacing"] = np.array(geom.detector_spacing)
        out[f"proj{ci}_rs"] = np.array(geom.source_to_origin or 0.0)
        out[f"proj{ci}_rd"] = np.array(geom.origin_to_detector or 0.0)
        out[f"proj{ci}_vol"] = vol
        out[f"proj{ci}_sino"] = sino.views.copy()
        out[f"proj{ci}_ys"] = ys
        out[f"proj{ci}_bp"] = bp.zyx.copy()
    out["proj_ncases"] = np.array(len(cases))


def gen_loss(out):
    rng = np.random.default_rng(7)
    cases = [(13, 17, 3), (5, 40, 2), (25, 96, 2), (12, 9, 1)]
    for ci, (m, n, p) in enumerate(cases):
        ref = rng.uniform(0, 3, (m, n, p)).astype(np.float32)
        pred = (ref + 0.3 * rng.standard_normal((m, n, p))).astype(np.float32)
        pred[0, 0, 0] = ref[0, 0, 0]  # an exact tie for the L1 sign
        vol = rng.uniform(0, 1, (4, 5, 6)).astype(np.float32)
        vol[0, 0, :2] = 0.25  # TV ties
        ps, rs = core.Sinogram.from_views(pred), core.Sinogram.from_views(ref)
        vg = core.VolumeGrid.from_zyx(vol)
        l1v, l1g = loss.l1_loss(ps, rs)
        sv, sg = loss.ssim_loss(ps, rs)
        tvv, tvg = loss.tv_loss(vg)
        tot, gp, gv, parts = loss.total_loss_detailed(ps, rs, vg, loss.LossWeights())
        for k, v in dict(pred=pred, ref=ref, vol=vol, l1=l1v, l1_grad=l1g, ssim=sv,
                         ssim_grad=sg, tv=tvv, tv_grad=tvg, total=tot, grad_pred=gp,
                         grad_vol=gv).items():
            out[f"loss{ci}_{k}"] = np.asarray(v)
    out["loss_ncases"] = np.array(len(cases))


def gen_adam(out):
    rng = np.random.default_rng(5)
    n = 37
    cl = core.GaussianCloud(rng.uniform(0, 30, (n, 3)), rng.uniform(0.2, 60, n),
                            rng.uniform(-0.001, 1, n).clip(0))
    g = core.ParamGradients(rng.standard_normal((n, 3)), rng.standard_normal(n),
                            rng.standard_normal(n), np.zeros(n), 1)
    st = optim.OptimizerState.fresh(n, 3e-4, 3e-5, 100)
    st = optim.OptimizerState(rng.standard_normal((n, 3)) * 0.1, rng.uniform(0, 0.1, (n, 3)),
                              rng.standard_normal(n) * 0.1, rng.uniform(0, 0.1, n),
                              rng.standard_normal(n) * 0.1, rng.uniform(0, 0.1, n), 17,
                              3e-4, 3e-5, 100)
    c2, s2 = optim.adam_step(cl, g, st, sigma_ceiling=51.0)
    for k, v in cloud_arrays(cl).items():
        out[f"adam_in_{k}"] = v
    for k in ("d_mu", "d_sigma", "d_intensity"):
        out[f"adam_{k}"] = np.array(getattr(g, k))
    for k in ("m_mu", "v_mu", "m_sigma", "v_sigma", "m_intensity", "v_intensity"):
        out[f"adam_in_{k}"] = np.array(getattr(st, k))
        out[f"adam_out_{k}"] = np.array(getattr(s2, k))
    out["adam_step"] = np.array(st.step)
    for k, v in cloud_arrays(c2).items():
        out[f"adam_out_{k}"] = v


# (n, n_max offset or None, grad_prune, tau, theta, box) per case; budgets:
# unlimited, clone-limited, split-limited, negative budget, sigma pruning
DENSIFY_CASES = [
    (400, None, True, 2e-4, 1.0, 17),
    (400, 10, True, 2e-4, 1.0, 17),
    (400, "split", True, 2e-4, 1.0, 17),
    (300, -5, False, 2e-4, 1.2, 5),
    (500, None, False, 1e-3, 0.8, 3),
]


def gen_densify(out):
    for ci, (n, nmax, gp, tau, theta, box) in enumerate(DENSIFY_CASES):
        rng = np.random.default_rng(100 + ci)
        mu = rng.uniform(-5, 70, (n, 3))
        sigma = rng.uniform(0.3, 4.0 * box if ci >= 3 else 3.0, n)
        inten = rng.uniform(0.0, 1.0, n)
        iters = int(rng.integers(1, 120))
        # avg spans tau: about a third below, the rest above (distinct values)
        accum = np.exp(rng.uniform(np.log(tau) - 2.0, np.log(tau) + 3.0, n)) * iters
        cl = core.GaussianCloud(mu, sigma, inten)
        g = core.ParamGradients(np.zeros((n, 3)), np.zeros(n), np.zeros(n), accum, iters)
        hot = (accum / iters >= tau)
        if nmax == "split":
            n_clone = int((hot & (sigma <= theta)).sum())
            n_max = n + n_clone + 7
        elif nmax is None:
            n_max = 10 * n
        else:
            n_max = n + nmax
        prm = densify.DensifyParams(n_max=n_max, tau=tau, theta=theta, box_size=box,
                                    grad_prune_enabled=gp)
        seed, it = 7 + ci, 100 * (ci + 1)
        new, rep = densify.densify_and_prune(cl, g, prm, np.random.default_rng([seed, it]))
        st = optim.OptimizerState(rng.standard_normal((n, 3)), rng.uniform(0, 1, (n, 3)),
                                  rng.standard_normal(n), rng.uniform(0, 1, n),
                                  rng.standard_normal(n), rng.uniform(0, 1, n), 5, 3e-4, 3e-5, 100)
        st2 = st.remap(rep)
        pre = f"d{ci}_"
        for k, v in dict(mu=mu, sigma=sigma, intensity=inten, accum=accum, iters=iters,
                         n_max=n_max, grad_prune=int(gp), tau=tau, theta=theta, box=box,
                         seed=seed, it=it).items():
            out[pre + k] = np.asarray(v)
        for k, v in cloud_arrays(new).items():
            out[pre + "out_" + k] = v
        out[pre + "report"] = np.array([rep.clones, rep.splits, rep.prunes, rep.n_after])
        out[pre + "kept"] = np.asarray(rep.kept)
        for k in ("m_mu", "v_mu", "m_sigma", "v_sigma", "m_intensity", "v_intensity"):
            out[pre + "in_" + k] = np.array(getattr(st, k))
            out[pre + "out_" + k] = np.array(getattr(st2, k))
        print(f"densify case {ci}: n {n} -> {rep.n_after} (clones {rep.clones}, "
              f"splits {rep.splits}, prunes {rep.prunes})")
    out["d_ncases"] = np.array(len(DENSIFY_CASES))


def c1_problem():
    dims = (64, 64, 64)
    truth = phantom.shepp_logan_3d(*dims)
    geom = core.ScanGeometry.parallel(25, 96)
    meas = projector.forward_project(truth, geom)
    return dims, truth, geom, meas


def gen_traj(out, iters=500):
    dims, truth, geom, meas = c1_problem()
    box = core.BoxConfig.for_dims(17, dims)
    base = projector.fbp(meas, geom, dims)
    init = optim.init_cloud_fbp(base, 10_000, 0, box=box)
    settings = optim.ReconstructionSettings(
        dims=dims, box=box, max_iters=iters, n_gaussians=10_000, seed=0,
        deterministic=True, densify_interval=0)
    t0 = time.time()
    vol, cloud, trace = optim.run_reconstruction(meas, geom, settings, truth=truth,
                                                 init_cloud=init)
    dt = time.time() - t0
    rep = metrics.volume_metrics(vol, truth)
    out["traj_iters"] = np.array(iters)
    out["traj_truth"] = truth.zyx.copy()
    out["traj_meas"] = meas.views.copy()
    out["traj_fbp"] = base.zyx.copy()
    for k, v in cloud_arrays(init).items():
        out[f"traj_init_{k}"] = v
    for k, v in cloud_arrays(cloud).items():
        out[f"traj_final_{k}"] = v
    out["traj_loss"] = np.array([r.loss for r in trace])
    out["traj_l1"] = np.array([r.loss_l1 for r in trace])
    out["traj_ssim"] = np.array([r.loss_ssim for r in trace])
    out["traj_tv"] = np.array([r.loss_tv for r in trace])
    out["traj_psnr"] = np.array([r.psnr for r in trace])
    out["traj_final_vol"] = vol.zyx.copy()
    out["traj_metrics"] = np.array([rep["psnr_volume"], rep["ssim_volume"]])
    out["traj_seconds"] = np.array(dt)
    print(f"traj: {iters} iters in {dt:.1f}s, final loss {trace[-1].loss:.6f}, "
          f"psnr {rep['psnr_volume']:.4f}, ssim {rep['ssim_volume']:.4f}")


def gen_c2pins(out, iters=4, n=50_000, n_samples=8192):
    """SURVEY 8(c) C2/C3 short pins, run by the reference itself.

    The 64 MB volumes and 26 MB sinograms are too big to commit; the fixture
    keeps the init clouds (the GPU test starts from exactly these), the full
    loss trace, the per-iteration parameter updates and seeded samples /
    norms of the measured sinogram, the FBP, and the final volume."""
    dims = (256, 256, 256)
    truth = phantom.shepp_logan_3d(*dims)
    box = core.BoxConfig.for_dims(17, dims)
    rng = np.random.default_rng(2024)
    vidx = rng.integers(0, 256 ** 3, n_samples)
    out["c2p_iters"] = np.array(iters)
    out["c2p_vol_idx"] = vidx
    out["c2p_truth_sum"] = np.array(truth.zyx.astype(np.float64).sum())
    for views in (50, 25):
        pre = f"c2p{views}_"
        geom = core.ScanGeometry.fan(views, 512, 1.6, 512.0, 512.0)
        t0 = time.time()
        meas = projector.forward_project(truth, geom)
        base = projector.fbp(meas, geom, dims)
        init = optim.init_cloud_fbp(base, n, 0, box=box)
        settings = optim.ReconstructionSettings(
            dims=dims, box=box, max_iters=iters, n_gaussians=n, seed=0,
            deterministic=True, densify_interval=0)
        vol, cloud, trace = optim.run_reconstruction(meas, geom, settings, init_cloud=init)
        dt = time.time() - t0
        # the same loop body (optim.py:350-403) spelled out with the reference's
        # own calls, to also keep the last iteration's parameter gradients
        c2, grads = init, None
        state = optim.OptimizerState.fresh(n, settings.lr_initial, settings.lr_final, iters)
        v2 = fvr.reconstruct(c2, box, dims, True)
        for it in range(iters):
            pred = projector.forward_project(v2, geom)
            value, g_pred, g_tv, _ = loss.total_loss_detailed(pred, meas, v2, settings.weights)
            assert value == trace[it].loss, (it, value, trace[it].loss)
            dg = projector.back_project(core.Sinogram.from_views(g_pred), geom, dims,
                                        deterministic=True).zyx.astype(np.float64)
            grads = fvr.backward(c2, box, dims, core.VolumeGrid.from_zyx(dg + g_tv), prev=grads)
            if it == 0:   # the init cloud's gradient: independent of the Adam path
                out[pre + "first_d_mu"] = np.array(grads.d_mu).astype(np.float32)
                out[pre + "first_d_sigma"] = np.array(grads.d_sigma).astype(np.float32)
                out[pre + "first_d_intensity"] = np.array(grads.d_intensity).astype(np.float32)
            c2, state = optim.adam_step(c2, grads, state, 3.0 * box.extent)
            v2 = fvr.reconstruct(c2, box, dims, True)
        assert np.array_equal(np.array(c2.mu), np.array(cloud.mu))
        out[pre + "last_d_mu"] = np.array(grads.d_mu).astype(np.float32)
        out[pre + "last_d_sigma"] = np.array(grads.d_sigma).astype(np.float32)
        out[pre + "last_d_intensity"] = np.array(grads.d_intensity).astype(np.float32)
        out[pre + "accum"] = np.array(grads.accum_pos_grad_norm).astype(np.float32)
        mv = meas.views
        sidx = rng.integers(0, mv.size, n_samples)
        out[pre + "meas_idx"] = sidx
        out[pre + "meas_samples"] = mv.reshape(-1)[sidx].copy()
        out[pre + "meas_norm"] = np.array(np.linalg.norm(mv.astype(np.float64)))
        out[pre + "fbp_samples"] = base.zyx.reshape(-1)[vidx].copy()
        out[pre + "fbp_norm"] = np.array(np.linalg.norm(base.zyx.astype(np.float64)))
        for k, v in cloud_arrays(init).items():
            out[pre + "init_" + k] = v
        fin = cloud_arrays(cloud)
        for k, v in cloud_arrays(init).items():
            out[pre + "delta_" + k] = fin[k] - v
        out[pre + "loss"] = np.array([r.loss for r in trace])
        out[pre + "l1"] = np.array([r.loss_l1 for r in trace])
        out[pre + "ssim"] = np.array([r.loss_ssim for r in trace])
        out[pre + "tv"] = np.array([r.loss_tv for r in trace])
        z = vol.zyx.astype(np.float64)
        out[pre + "vol_samples"] = vol.zyx.reshape(-1)[vidx].copy()
        out[pre + "vol_norm"] = np.array(np.linalg.norm(z))
        out[pre + "vol_sum"] = np.array(z.sum())
        out[pre + "seconds"] = np.array(dt)
        print(f"c2pins {views} views: losses {[round(r.loss, 6) for r in trace]} ({dt:.0f} s)")


API_NAMES = [
    ("core", "GaussianCloud"), ("core", "BoxConfig.cube"), ("core", "BoxConfig.for_dims"),
    ("core", "VolumeGrid.from_zyx"), ("core", "Sinogram.from_views"),
    ("core", "ScanGeometry.parallel"), ("core", "ScanGeometry.fan"), ("core", "ParamGradients"),
    ("core", "make_offset_grid"), ("core", "validate_cloud"),
    ("fvr", "reconstruct"), ("fvr", "reconstruct_nodecomp"), ("fvr", "reconstruct_direct"),
    ("fvr", "backward"),
    ("projector", "forward_project"), ("projector", "back_project"), ("projector", "fbp"),
    ("loss", "l1_loss"), ("loss", "ssim_loss"), ("loss", "tv_loss"), ("loss", "total_loss"),
    ("loss", "total_loss_detailed"), ("loss", "ssim_value"), ("loss", "LossWeights"),
    ("optim", "adam_step"), ("optim", "OptimizerState.fresh"), ("optim", "init_cloud_fbp"),
    ("optim", "init_cloud_random"), ("optim", "run_reconstruction"),
    ("optim", "ReconstructionSettings"),
    ("densify", "densify_and_prune"), ("metrics", "psnr"), ("metrics", "volume_metrics"),
    ("phantom", "shepp_logan_3d"),
]


def gen_api():
    """Public names and call signatures of the reference package (the drop-in
    boundary): parameter names, kinds and which have defaults."""
    import importlib
    import inspect
    import json
    out = {"__all__": list(splatct.__all__), "signatures": {}}
    for mod, qual in API_NAMES:
        obj = importlib.import_module(f"splatct.{mod}")
        for part in qual.split("."):
            obj = getattr(obj, part)
        sig = inspect.signature(obj)
        out["signatures"][f"{mod}.{qual}"] = [
            [p.name, p.kind.name, p.default is not inspect.Parameter.empty]
            for p in sig.parameters.values()]
    with open(os.path.join(HERE, "api_signatures.json"), "w") as f:
        json.dump(out, f, indent=1)
    print("wrote api_signatures.json with", len(out["signatures"]), "signatures")


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--traj", action="store_true")
    ap.add_argument("--only", choices=["densify", "c2pins", "api"], default=None)
    args = ap.parse_args()
    if args.only == "api":
        gen_api()
        return
    if args.only == "c2pins":
        d = {}
        gen_c2pins(d)
        d["versions"] = np.array(
            f"numpy {np.__version__}; scipy {__import__('scipy').__version__}; "
            f"numba {__import__('numba').__version__}")
        np.savez_compressed(os.path.join(HERE, "c2pins.npz"), **d)
        print("wrote c2pins.npz with", len(d), "arrays")
        return
    d = {}
    gen_densify(d)
    np.savez_compressed(os.path.join(HERE, "densify.npz"), **d)
    print("wrote densify.npz with", len(d), "arrays")
    if args.only == "densify":
        return
    out = {}
    gen_fvr(out)
    gen_proj(out)
    gen_loss(out)
    gen_adam(out)
    out["versions"] = np.array(
        f"numpy {np.__version__}; scipy {__import__('scipy').__version__}; "
        f"numba {__import__('numba').__version__}")
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **out)
    print("wrote kernels.npz with", len(out), "arrays")
    if args.traj:
        t = {}
        gen_traj(t)
        np.savez_compressed(os.path.join(HERE, "traj_c1.npz"), **t)
        print("wrote traj_c1.npz")


if __name__ == "__main__":
    main()
