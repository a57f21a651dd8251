"""Parity of the B200 path (libsplatct via the product API) against the
reference's golden vectors and the CPU oracle.  Tolerances (BASELINE.json
north_star): footprints and tile bin lists bit-exact; volumes and
projections <= 1e-5 relative L2; parameter gradients <= 1e-4 relative L2;
final PSNR within 0.05 dB of the reference after a fixed iteration count.
"""
import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_2411_04844_b200 import core, densify, device as D, fvr, loss, metrics, optim, phantom, projector  # noqa: E402
from paper_2411_04844_b200.trainer import Trainer  # noqa: E402

VOL_TOL = 1e-5
GRAD_TOL = 1e-4


def _cloud(g, pfx):
    return core.GaussianCloud(g[f"{pfx}_mu"], g[f"{pfx}_sigma"], g[f"{pfx}_intensity"])


def _geom(g, ci):
    p = lambda k: g[f"proj{ci}_{k}"]
    ang = p("angles")
    if str(p("variant")) == "fan":
        return core.ScanGeometry("fan", len(ang), int(p("n_det")), float(p("spacing")), ang,
                                 float(p("rs")), float(p("rd")))
    return core.ScanGeometry("parallel", len(ang), int(p("n_det")), float(p("spacing")), ang)


# --------------------------------------------------------------------------- voxelizer
@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_fvr_forward_golden(kernels_golden):
    g = kernels_golden
    for ci in range(int(g["fvr_ncases"])):
        dims = tuple(int(v) for v in g[f"fvr{ci}_dims"])
        box = core.BoxConfig(*(int(v) for v in g[f"fvr{ci}_box"]))
        vol = fvr.reconstruct(_cloud(g, f"fvr{ci}"), box, dims)
        ref = g[f"fvr{ci}_vol"]
        assert rel_l2(vol.zyx, ref) < VOL_TOL, ci
        assert np.abs(vol.zyx - ref).max() < 1e-5 * max(1.0, np.abs(ref).max())


def test_spec_single_gaussian(kernels_golden):
    box = core.BoxConfig.cube(17)
    v = fvr.reconstruct(core.GaussianCloud([[8.0, 8, 8]], [1.0], [1.0]), box, (17, 17, 17))
    assert v.at(8, 8, 8) == 1.0 and abs(v.at(9, 8, 8) - np.exp(-0.5)) < 1e-7
    v = fvr.reconstruct(core.GaussianCloud([[8.5, 8, 8]], [1.0], [1.0]), box, (17, 17, 17))
    assert abs(v.at(8, 8, 8) - np.exp(-0.125)) < 1e-7 and v.at(8, 8, 8) == v.at(9, 8, 8)


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_fvr_bins_bit_exact(kernels_golden):
    g = kernels_golden
    dev = D.require_cuda()
    rng = np.random.default_rng(11)
    cases = []
    for ci in range(int(g["fvr_ncases"])):
        cases.append((g[f"fvr{ci}_mu"], tuple(int(v) for v in g[f"fvr{ci}_dims"]),
                      tuple(int(v) for v in g[f"fvr{ci}_box"])))
    mu = rng.uniform(-10, 140, (20000, 3))
    mu[:50] = np.floor(mu[:50])          # exact integers
    mu[50:60] = -1e-12                   # floor -> -1
    cases.append((mu, (128, 96, 130), (17, 17, 17)))
    for mu, dims, box in cases:
        n = mu.shape[0]
        params = torch.zeros((5, n), dtype=torch.float64, device=dev)
        params[0:3] = torch.from_numpy(np.ascontiguousarray(mu.T)).to(dev)
        params[3] = 1.0
        plan = D.FvrPlan(n, dims, O.box_half(box), 0, dev)
        plan.bin(params)
        fp, ts, items = plan.export_bins()
        ofp, ots, oitems = O.bins(mu, box, dims, (16, 16, 16))
        np.testing.assert_array_equal(fp, ofp)
        np.testing.assert_array_equal(ts.astype(np.int64), ots)
        np.testing.assert_array_equal(items, oitems)


@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_fvr_backward_golden(kernels_golden):
    g = kernels_golden
    for ci in range(int(g["fvr_ncases"])):
        dims = tuple(int(v) for v in g[f"fvr{ci}_dims"])
        box = core.BoxConfig(*(int(v) for v in g[f"fvr{ci}_box"]))
        up = core.VolumeGrid.from_zyx(g[f"fvr{ci}_up"])
        gr = fvr.backward(_cloud(g, f"fvr{ci}"), box, dims, up)
        assert rel_l2(gr.d_mu, g[f"fvr{ci}_d_mu"]) < GRAD_TOL, ci
        assert rel_l2(gr.d_sigma, g[f"fvr{ci}_d_sigma"]) < GRAD_TOL, ci
        assert rel_l2(gr.d_intensity, g[f"fvr{ci}_d_intensity"]) < GRAD_TOL, ci
        assert rel_l2(gr.accum_pos_grad_norm, g[f"fvr{ci}_accum"]) < GRAD_TOL, ci
        assert gr.iters_since_densify == 1


@pytest.mark.parametrize("dims,n,clustered", [((128, 128, 128), 50_000, False),
                                              ((96, 80, 64), 20_000, True)])
def test_fvr_vs_oracle_sweep_point(dims, n, clustered):
    """A voxelize-sweep point against the oracle: fwd + bwd."""
    rng = np.random.default_rng(0)
    box = core.BoxConfig.for_dims(17, dims)
    if clustered:
        c = np.array(dims) / 2
        mu = c + rng.standard_normal((n, 3)) * np.array(dims) / 8
        sig = rng.uniform(0.5, 3.0, n)
        inten = rng.uniform(0, 1, n)
    else:
        cl = optim.init_cloud_random(dims, n, seed=0, box=box)
        mu, sig, inten = cl.mu, cl.sigma, cl.intensity
    cloud = core.GaussianCloud(mu, sig, inten)
    vol = fvr.reconstruct(cloud, box, dims)
    ovol = O.splat_fwd(mu, sig, inten, box.shape, dims)
    assert rel_l2(vol.zyx, ovol) < VOL_TOL
    up = rng.standard_normal(dims[::-1]).astype(np.float32)
    gr = fvr.backward(cloud, box, dims, core.VolumeGrid.from_zyx(up))
    dm, ds, di, _, _ = O.splat_bwd(mu, sig, inten, box.shape, dims, up)
    assert rel_l2(gr.d_mu, dm) < GRAD_TOL
    assert rel_l2(gr.d_sigma, ds) < GRAD_TOL
    assert rel_l2(gr.d_intensity, di) < GRAD_TOL


def test_fvr_deterministic_and_direct():
    rng = np.random.default_rng(4)
    dims = (32, 32, 32)
    cl = core.GaussianCloud(rng.uniform(8, 24, (20, 3)), rng.uniform(0.5, 1.5, 20),
                            rng.uniform(0, 1, 20))
    box = core.BoxConfig.cube(17)
    a = fvr.reconstruct(cl, box, dims).zyx
    b = fvr.reconstruct(cl, box, dims).zyx
    np.testing.assert_array_equal(a, b)
    c = fvr.reconstruct_direct(cl, dims).zyx
    assert np.abs(a - c).max() <= 1e-4 * np.abs(c).max()
    ref = O.splat_direct(cl.mu, cl.sigma, cl.intensity, dims)
    assert rel_l2(c, ref) < VOL_TOL


# --------------------------------------------------------------------------- projector
def test_projector_golden(kernels_golden):
    g = kernels_golden
    for ci in range(int(g["proj_ncases"])):
        geom = _geom(g, ci)
        dims = tuple(int(v) for v in g[f"proj{ci}_dims"])
        s = projector.forward_project(core.VolumeGrid.from_zyx(g[f"proj{ci}_vol"]), geom)
        assert rel_l2(s.views, g[f"proj{ci}_sino"]) < VOL_TOL, ci
        bp = projector.back_project(core.Sinogram.from_views(g[f"proj{ci}_ys"]), geom, dims)
        assert rel_l2(bp.zyx, g[f"proj{ci}_bp"]) < VOL_TOL, ci


@pytest.mark.parametrize("variant", ["parallel", "fan"])
def test_projector_dot_test_and_march(variant):
    dev = D.require_cuda()
    w, h, c = 64, 64, 8
    geom = (core.ScanGeometry.parallel(30, 90) if variant == "parallel"
            else core.ScanGeometry.fan(30, 120, 1.3, 80.0, 60.0))
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    g = torch.Generator(device="cpu").manual_seed(0)
    x = torch.randn((h, w, c), generator=g).to(dev)
    y = torch.randn((30, geom.n_detectors, c), generator=g).to(dev)
    ax = op.forward(x)
    aty = op.adjoint(y)
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    assert abs(lhs - rhs) / abs(lhs) < 1e-5
    assert rel_l2(op.march_forward(x).cpu().numpy(), ax.cpu().numpy()) < 1e-6


def test_projector_c2_geometry_vs_oracle():
    """The headline geometry (fan 50 x 512, 256^2 slices) against the oracle."""
    dev = D.require_cuda()
    geom = core.ScanGeometry.fan(50, 512, 1.6, 512.0, 512.0)
    ogeom = O.Geometry.fan(50, 512, 1.6, 512.0, 512.0)
    rng = np.random.default_rng(1)
    vol = rng.uniform(0, 1, (4, 256, 256)).astype(np.float32)
    s = projector.forward_project(core.VolumeGrid.from_zyx(vol), geom)
    assert rel_l2(s.views, O.project_forward(vol, ogeom)) < VOL_TOL
    ys = rng.standard_normal((50, 512, 4)).astype(np.float32)
    bp = projector.back_project(core.Sinogram.from_views(ys), geom, (256, 256, 4))
    assert rel_l2(bp.zyx, O.project_adjoint(ys, ogeom, (256, 256, 4))) < VOL_TOL


def test_disk_chord():
    """central parallel ray through a disk of radius R gives ~2R."""
    n = 128
    yy, xx = np.mgrid[0:n, 0:n]
    disk = (((xx - 63.5) ** 2 + (yy - 63.5) ** 2) <= 40 ** 2).astype(np.float32)[None]
    s = projector.forward_project(core.VolumeGrid.from_zyx(disk), core.ScanGeometry.parallel(4, 129))
    assert abs(s.views[0, 64, 0] - 80.0) / 80.0 < 0.02


# --------------------------------------------------------------------------- loss + adam
def test_loss_golden(kernels_golden):
    g = kernels_golden
    for ci in range(int(g["loss_ncases"])):
        p = lambda k: g[f"loss{ci}_{k}"]
        pred, ref = core.Sinogram.from_views(p("pred")), core.Sinogram.from_views(p("ref"))
        vol = core.VolumeGrid.from_zyx(p("vol"))
        v, gp, gv, parts = loss.total_loss_detailed(pred, ref, vol, loss.LossWeights())
        assert abs(v - float(p("total"))) < 1e-9, ci
        assert abs(parts["l1"] - float(p("l1"))) < 1e-12
        assert abs(parts["ssim"] - float(p("ssim"))) < 1e-9
        assert abs(parts["tv"] - float(p("tv"))) < 1e-12
        assert rel_l2(gp, p("grad_pred")) < 1e-6, ci
        assert rel_l2(gv, p("grad_vol")) < 1e-6, ci
        sv, sg = loss.ssim_loss(pred, ref)
        assert abs(sv - float(p("ssim"))) < 1e-9 and rel_l2(sg, p("ssim_grad")) < 1e-6


def test_ssim_value_and_psnr():
    rng = np.random.default_rng(2)
    x = rng.uniform(0, 1, (40, 30))
    assert abs(loss.ssim_value(x, x) - 1.0) < 1e-9
    y = rng.uniform(0, 1, (40, 30))
    # images enter the kernels as float32 (the training loop's storage type)
    assert abs(loss.ssim_value(x, y) - O.ssim_value(x, y)) < 1e-6
    xf, yf = x.astype(np.float32), y.astype(np.float32)
    assert abs(loss.ssim_value(xf, yf) - O.ssim_value(xf, yf)) < 1e-12
    assert metrics.psnr(np.full(10, 0.1), np.zeros(10), max_val=1.0) == pytest.approx(20.0, abs=1e-12)


def test_adam_golden(kernels_golden):
    g = kernels_golden
    cl = core.GaussianCloud(g["adam_in_mu"], g["adam_in_sigma"], g["adam_in_intensity"])
    gr = core.ParamGradients(g["adam_d_mu"], g["adam_d_sigma"], g["adam_d_intensity"],
                             np.zeros(len(g["adam_d_sigma"])), 1)
    st = optim.OptimizerState(*(g[f"adam_in_{k}"] for k in ("m_mu", "v_mu", "m_sigma", "v_sigma",
                                                             "m_intensity", "v_intensity")),
                              int(g["adam_step"]), 3e-4, 3e-5, 100)
    c2, s2 = optim.adam_step(cl, gr, st, 51.0)
    np.testing.assert_allclose(c2.mu, g["adam_out_mu"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(c2.sigma, g["adam_out_sigma"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(c2.intensity, g["adam_out_intensity"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(s2.v_mu, g["adam_out_v_mu"], rtol=1e-14)
    assert s2.step == int(g["adam_step"]) + 1


# --------------------------------------------------------------------------- FBP + init
def test_fbp_and_init_cloud(traj_golden):
    g = traj_golden
    geom = core.ScanGeometry.parallel(25, 96)
    meas = core.Sinogram.from_views(g["traj_meas"])
    vol = projector.fbp(meas, geom, (64, 64, 64))
    assert rel_l2(vol.zyx, g["traj_fbp"]) < 1e-6
    cl = optim.init_cloud_fbp(vol, 10_000, 0, box=core.BoxConfig.for_dims(17, (64, 64, 64)))
    same = np.all(cl.mu == g["traj_init_mu"], axis=1).mean()
    assert same > 0.999
    assert rel_l2(cl.intensity, g["traj_init_intensity"]) < 1e-3


# --------------------------------------------------------------------------- z-slab emulation
def test_slab_emulation_matches_full():
    """Voxelizer + TV-fused adjoint on G z-slabs of one device match unsharded (fp32 rounding)."""
    dev = D.require_cuda()
    dims = (48, 40, 64)
    w, h, c = dims
    box = core.BoxConfig.cube(17)
    cl = optim.init_cloud_random(dims, 3000, seed=5, box=box)
    params = D.cloud_to_params(cl, dev)
    full = D.FvrPlan(cl.n, dims, box.half, 0, dev)
    vfull = full.new_volume()
    full.bin(params)
    full.forward(params, vfull)
    rng = torch.Generator().manual_seed(3)
    up = torch.randn((h, w, c), generator=rng).to(dev)
    gfull = torch.empty((5, cl.n), dtype=torch.float64, device=dev)
    full.backward(params, up, gfull)
    geom = core.ScanGeometry.parallel(20, 70)
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    gs = torch.randn((20, 70, c), generator=rng).to(dev)
    dl_full = op.adjoint(gs, vol=vfull, lambda_tv=0.7, tv_count=float(w * h * c))
    from paper_2411_04844_b200.distributed import slab_bounds
    G = 3
    gsum = torch.zeros_like(gfull)
    for r in range(G):
        s = slab_bounds(c, G, r)
        plan = D.FvrPlan(cl.n, (w, h, s.c_local), box.half, s.z0, dev)
        v = plan.new_volume()
        plan.bin(params)
        plan.forward(params, v)
        # slab tiles group Gaussians into different tensor-core k8 steps than
        # the full volume's tiles, so sums agree to fp32 rounding, not bitwise
        assert rel_l2(v.cpu().numpy(), vfull[:, :, s.z0:s.z0 + s.c_local].cpu().numpy()) < 1e-6
        gl = torch.empty_like(gfull)
        plan.backward(params, up[:, :, s.z0:s.z0 + s.c_local].contiguous(), gl)
        gsum += gl
        lo = vfull[:, :, s.z0 - 1].contiguous() if s.z0 > 0 else None
        hi = vfull[:, :, s.z0 + s.c_local].contiguous() if s.z0 + s.c_local < c else None
        dl = op.adjoint(gs[:, :, s.z0:s.z0 + s.c_local].contiguous(), vol=v, halo_lo=lo,
                        halo_hi=hi, lambda_tv=0.7, tv_count=float(w * h * c))
        assert rel_l2(dl.cpu().numpy(), dl_full[:, :, s.z0:s.z0 + s.c_local].cpu().numpy()) < 1e-6
    assert rel_l2(gsum.cpu().numpy(), gfull.cpu().numpy()) < 1e-6


# --------------------------------------------------------------------------- training
def test_trainer_matches_oracle_iterations(traj_golden):
    """Eight device iterations vs the oracle loop on config 1 (loss trace)."""
    g = traj_golden
    dev = D.require_cuda()
    dims = (64, 64, 64)
    box = core.BoxConfig.for_dims(17, dims)
    geom = core.ScanGeometry.parallel(25, 96)
    cl = core.GaussianCloud(g["traj_init_mu"], g["traj_init_sigma"], g["traj_init_intensity"])
    tr = Trainer(D.sino_to_device(g["traj_meas"], dev), geom, dims, box, loss.LossWeights(),
                 D.cloud_to_params(cl, dev), max_iters=500, trace_cap=8)
    tr.initial_volume()
    for _ in range(8):
        tr.step()
    rows = tr.trace_rows()
    assert rows.shape[0] == 8
    np.testing.assert_allclose(rows[:, 0], g["traj_loss"][:8], rtol=2e-6)


@pytest.mark.slow
def test_trajectory_c1_psnr(traj_golden):
    """Config 1, 500 iterations (graph-replayed): PSNR within 0.05 dB of the reference."""
    g = traj_golden
    dims = (64, 64, 64)
    box = core.BoxConfig.for_dims(17, dims)
    geom = core.ScanGeometry.parallel(25, 96)
    cl = core.GaussianCloud(g["traj_init_mu"], g["traj_init_sigma"], g["traj_init_intensity"])
    settings = optim.ReconstructionSettings(dims=dims, box=box, max_iters=500, n_gaussians=10_000,
                                            seed=0, deterministic=True, densify_interval=0)
    vol, cloud, trace = optim.run_reconstruction(core.Sinogram.from_views(g["traj_meas"]), geom,
                                                 settings, init_cloud=cl)
    assert len(trace) == 500 and trace[-1].iteration == 500
    losses = np.array([r.loss for r in trace])
    assert np.all(np.isfinite(losses))
    np.testing.assert_allclose(losses[[0, 100, 200, 300, 400, 499]],
                               g["traj_loss"][[0, 100, 200, 300, 400, 499]], rtol=1e-3)
    truth = core.VolumeGrid.from_zyx(g["traj_truth"])
    rep = metrics.volume_metrics(vol, truth)
    ref_psnr, ref_ssim = (float(v) for v in g["traj_metrics"])
    assert abs(rep["psnr_volume"] - ref_psnr) <= 0.05
    assert rep["ssim_volume"] >= 0.9 * ref_ssim


def test_run_reconstruction_eager_paths():
    """truth metrics, densification and the val stop rule (host events per iteration)."""
    dims = (32, 32, 32)
    truth = phantom.shepp_logan_3d(32, 32, 32)
    geom = core.ScanGeometry.parallel(12, 48)
    meas = projector.forward_project(truth, geom)
    box = core.BoxConfig.for_dims(17, dims)
    st = optim.ReconstructionSettings(dims=dims, box=box, max_iters=6, n_gaussians=800,
                                      densify_interval=3, init_mode="fbp",
                                      densify=densify.DensifyParams(grad_prune_enabled=False,
                                                                    tau=1e-12))
    vol, cl, trace = optim.run_reconstruction(meas, geom, st, truth=truth)
    assert [r.iteration for r in trace] == list(range(1, 7))
    assert all(np.isfinite(r.psnr) and np.isfinite(r.ssim) for r in trace)
    assert trace[2].clones + trace[2].splits > 0 and cl.n == trace[-1].n_gaussians
    st2 = optim.ReconstructionSettings(dims=dims, box=box, max_iters=5, n_gaussians=500,
                                       densify_interval=0, stop_rule="val-convergence",
                                       patience=2)
    _, _, tr2 = optim.run_reconstruction(meas, geom, st2)
    assert all(np.isfinite(r.val_loss) for r in tr2)


def test_nonfinite_loss_raises():
    dims = (32, 32, 32)
    geom = core.ScanGeometry.parallel(8, 48)
    meas = core.Sinogram.from_views(np.ones((8, 48, 32), np.float32))
    cl = core.GaussianCloud([[16.0, 16, 16]], [1.0], [1e300])   # inf once stored as f32
    st = optim.ReconstructionSettings(dims=dims, box=core.BoxConfig.cube(17), max_iters=3,
                                      densify_interval=0)
    with pytest.raises(optim.NonFiniteLossError) as ei:
        optim.run_reconstruction(meas, geom, st, init_cloud=cl)
    assert ei.value.snapshot["iteration"] == 0


@pytest.mark.parametrize("variant,dims,m,n", [("parallel", (24, 20, 70), 7, 30),
                                              ("fan", (13, 21, 300), 6, 17),
                                              ("fan", (64, 48, 5), 11, 93)])
def test_blocked_operator_matches_csr(variant, dims, m, n):
    """4-row blocked A / A^T (+TV epilogue) equal the CSR operators."""
    dev = D.require_cuda()
    w, h, c = dims
    geom = (core.ScanGeometry.parallel(m, n, 0.9) if variant == "parallel"
            else core.ScanGeometry.fan(m, n, 1.7, 60.0, 40.0))
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    g = torch.Generator().manual_seed(1)
    x = torch.randn((h, w, c), generator=g).to(dev)
    y = torch.randn((m, n, c), generator=g).to(dev)
    a = op.forward(x, blocked=True)
    b = op.forward(x, blocked=False)
    assert rel_l2(a.cpu().numpy(), b.cpu().numpy()) < 1e-6
    pa = torch.zeros(D.tv_partial_len(w, h, c), dtype=torch.float64, device=dev)
    pb = torch.zeros_like(pa)
    a = op.adjoint(y, vol=x, lambda_tv=0.3, tv_count=float(w * h * c), tv_partial=pa, blocked=True)
    b = op.adjoint(y, vol=x, lambda_tv=0.3, tv_count=float(w * h * c), tv_partial=pb, blocked=False)
    assert rel_l2(a.cpu().numpy(), b.cpu().numpy()) < 1e-6
    assert abs(float(pa.sum()) - float(pb.sum())) <= 1e-8 * abs(float(pb.sum()))


@pytest.mark.parametrize("dims,c_note", [((96, 80, 256), "c=256: two 128-z chunks"),
                                         ((64, 48, 40), "c=40: 32-z chunks, partial tile")])
def test_projector_occupancy_skip_is_exact(dims, c_note):
    """Empty-space skipping (voxelizer tile occupancy) changes nothing: a cloud
    confined to part of the volume, projected with and without the mask."""
    dev = D.require_cuda()
    w, h, c = dims
    rng = np.random.default_rng(12)
    n = 3000
    mu = np.stack([rng.uniform(10, w * 0.45, n), rng.uniform(5, h - 5, n),
                   rng.uniform(c * 0.2, c * 0.5, n)], 1)
    cloud = core.GaussianCloud(mu, rng.uniform(0.6, 2.0, n), rng.uniform(0, 1, n))
    box = core.BoxConfig.for_dims(17, dims)
    plan = D.FvrPlan(n, dims, box.half, 0, dev)
    params = D.cloud_to_params(cloud, dev)
    plan.bin(params)
    vol = plan.forward(params, plan.new_volume(), masks=True)
    occ = plan.pixel_occupancy_words().cpu().numpy().view(np.uint64)
    assert 0 < int(sum(bin(int(v)).count("1") for v in occ)) < occ.size * ((c + 15) // 16)
    geom = core.ScanGeometry.fan(20, 90, 1.3, 120.0, 90.0)
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    dense = op.forward(vol)
    skip = op.forward(vol, occ=plan)
    np.testing.assert_array_equal(skip.cpu().numpy(), dense.cpu().numpy())


def test_trainer_occupancy_skipping_is_exact():
    """The training step with empty-space skipping (projector forward entries,
    adjoint quads) equals the dense step bitwise: same loss trace and cloud
    after ten iterations on a phantom with empty space around the body."""
    dev = D.require_cuda()
    dims = (96, 96, 64)
    # a ball in a larger field of view: empty space around it
    zz, yy, xx = np.mgrid[0:64, 0:96, 0:96]
    ball = ((xx - 40.0) ** 2 + (yy - 52.0) ** 2 + (zz - 30.0) ** 2 <= 18.0 ** 2)
    truth = core.VolumeGrid.from_zyx(ball.astype(np.float32))
    geom = core.ScanGeometry.fan(30, 160, 1.0, 150.0, 110.0)
    meas = projector.forward_project(truth, geom)
    box = core.BoxConfig.for_dims(17, dims)
    rng = np.random.default_rng(13)
    n = 3000
    d = rng.normal(size=(n, 3))
    d *= (rng.uniform(0, 1, n) ** (1 / 3) * 15.0 / np.linalg.norm(d, axis=1))[:, None]
    cl = core.GaussianCloud(d + np.array([40.0, 52.0, 30.0]), np.full(n, 1.5),
                            np.full(n, 0.05))
    outs = []
    for skip in (True, False):
        tr = Trainer(D.sino_to_device(meas.views, dev), geom, dims, box, loss.LossWeights(),
                     D.cloud_to_params(cl, dev), max_iters=100, trace_cap=10)
        if not skip:
            tr.fvr.footprint_coverage = tr.fvr.pixel_occupancy = None
        tr.initial_volume()
        for _ in range(10):
            tr.step()
        if skip:   # the phantom leaves empty tiles, so the skipping paths run
            words = tr.fvr.footprint_coverage_words().cpu().numpy().view(np.uint64)
            assert sum(bin(int(v)).count("1") for v in words) < words.size * 4
        outs.append((tr.trace_rows().copy(), tr.params.cpu().numpy()))
    np.testing.assert_array_equal(outs[0][0], outs[1][0])
    np.testing.assert_array_equal(outs[0][1], outs[1][1])


# --------------------------------------------------------------------------- a7: non-decomposed
@pytest.mark.filterwarnings("ignore::RuntimeWarning")
def test_fvr_nodecomp_golden_and_oracle(kernels_golden):
    """fvr.reconstruct_nodecomp (splat_plain, _kernels.py:81-129) on the device:
    the reference's golden volumes and the oracle's splat_plain, <= 1e-5."""
    g = kernels_golden
    for ci in range(int(g["fvr_ncases"])):
        dims = tuple(int(v) for v in g[f"fvr{ci}_dims"])
        box = core.BoxConfig(*(int(v) for v in g[f"fvr{ci}_box"]))
        cl = _cloud(g, f"fvr{ci}")
        vol = fvr.reconstruct_nodecomp(cl, box, dims)
        assert rel_l2(vol.zyx, g[f"fvr{ci}_vol"]) < VOL_TOL, ci
        assert rel_l2(vol.zyx, O.splat_plain(cl.mu, cl.sigma, cl.intensity, box.shape, dims)) < VOL_TOL
    dims = (128, 128, 128)
    box = core.BoxConfig.for_dims(17, dims)
    cl = optim.init_cloud_random(dims, 20_000, seed=3, box=box)
    a = fvr.reconstruct_nodecomp(cl, box, dims).zyx
    assert rel_l2(a, O.splat_plain(cl.mu, cl.sigma, cl.intensity, box.shape, dims)) < VOL_TOL
    assert rel_l2(a, fvr.reconstruct(cl, box, dims).zyx) < VOL_TOL


def test_decomposition_speedup_spec():
    """at 50k Gaussians, a 17^3 box and a 128^3 grid the
    decomposed splat is >= 2x faster than the non-decomposed one (device
    times of the splat kernels on the same bins, CUDA events)."""
    dev = D.require_cuda()
    dims = (128, 128, 128)
    box = core.BoxConfig.for_dims(17, dims)
    cl = optim.init_cloud_random(dims, 50_000, seed=0, box=box)
    params = D.cloud_to_params(cl, dev)
    plan = D.FvrPlan(cl.n, dims, box.half, 0, dev)
    out = plan.new_volume()
    plan.bin(params)

    def med(fn, reps=7):
        fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(True), torch.cuda.Event(True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return sorted(ts)[reps // 2]

    t_dec = med(lambda: plan.forward(params, out))
    t_plain = med(lambda: plan.forward_plain(params, out))
    print(f"decomposed {t_dec:.3f} ms, non-decomposed {t_plain:.3f} ms, ratio {t_plain / t_dec:.2f}")
    assert t_plain >= 2.0 * t_dec
