"""Parity at BASELINE.json's full sizes, where the whole-problem oracle would
take minutes, through checks that do not depend on size:

- tile bins at C4 (512^3, 400k) and at the largest C5 point (1024^3, 2M):
  footprints, tile starts and per-tile Gaussian lists bit-exact against the
  CPU restatement (the north star's bit-exact requirement);
- voxelizer forward at C4: a 48^3 sub-block (interior and at the volume
  corner) against the oracle splat of the Gaussians whose boxes reach it --
  the floor of mu - o is floor(mu) - o for an integer offset o, so the
  oracle's clipping to the sub-block changes nothing inside it;
- voxelizer backward at C4: every Gaussian's gradient depends only on the
  upstream inside its box, so a random sample of 3000 Gaussians is checked
  against the oracle with the full 512^3 upstream;
- projector pair at C2 and C4 geometry: full-size adjoint dot test in f64,
  and sampled slices against the oracle (the per-slice operator reads only
  its own slice, _kernels.py:273-278);
- fused loss at the full C2 sinogram (50 x 512 x 256) against the oracle.
Tolerances as test_gpu_parity.py.
"""
import numpy as np
import pytest
import torch

from conftest import rel_l2
from oracle import oracle as O

pytestmark = pytest.mark.gpu

from paper_2411_04844_b200 import core, device as D, loss, optim  # noqa: E402

VOL_TOL = 1e-5
GRAD_TOL = 1e-4


def _params(cloud, dev):
    return D.cloud_to_params(cloud, dev)


@pytest.mark.parametrize("g,n", [(512, 400_000), (1024, 2_000_000)])
def test_bins_bit_exact_full_size(g, n):
    dev = D.require_cuda()
    dims = (g, g, g)
    box = core.BoxConfig.for_dims(17, dims)
    cloud = optim.init_cloud_random(dims, n, seed=0, box=box)
    plan = D.FvrPlan(n, dims, box.half, 0, dev)
    plan.bin(_params(cloud, dev))
    fp, ts, items = plan.export_bins()
    ofp, ots, oitems = O.bins(cloud.mu, box.shape, dims, (16, 16, 16))
    np.testing.assert_array_equal(fp, ofp)
    np.testing.assert_array_equal(ts.astype(np.int64), ots)
    np.testing.assert_array_equal(items, oitems)


def _c4_cloud():
    dims = (512, 512, 512)
    box = core.BoxConfig.for_dims(17, dims)
    rng = np.random.default_rng(4)
    n = 400_000
    # uniform centres incl. boxes clipped by the faces, sigma spread, f32-exact
    mu = rng.uniform(-6, 518, (n, 3)).astype(np.float32).astype(np.float64)
    sigma = rng.uniform(0.5, 3.0, n).astype(np.float32).astype(np.float64)
    inten = rng.uniform(0, 1, n).astype(np.float32).astype(np.float64)
    return dims, box, core.GaussianCloud(mu, sigma, inten)


@pytest.mark.filterwarnings("ignore:Gaussian centers outside the volume")
def test_fvr_forward_c4_subblocks():
    dev = D.require_cuda()
    dims, box, cloud = _c4_cloud()
    plan = D.FvrPlan(cloud.n, dims, box.half, 0, dev)
    params = _params(cloud, dev)
    plan.bin(params)
    vol = plan.forward(params, plan.new_volume())          # (h, w, c)
    hv = np.array(box.half, np.float64)
    b = 48
    for o in ((0, 0, 0), (231, 140, 300), (464, 464, 464)):
        o = np.array(o)
        fl = np.floor(cloud.mu)
        reach = np.all((fl + hv >= o) & (fl - hv < o + b), axis=1)
        sub = O.splat_fwd(cloud.mu[reach] - o, cloud.sigma[reach], cloud.intensity[reach],
                          box.shape, (b, b, b))        # (z, y, x)
        got = vol[o[1]:o[1] + b, o[0]:o[0] + b, o[2]:o[2] + b].permute(2, 0, 1).cpu().numpy()
        assert rel_l2(got, sub) < VOL_TOL, tuple(o)


@pytest.mark.filterwarnings("ignore:Gaussian centers outside the volume")
def test_fvr_backward_c4_sampled():
    dev = D.require_cuda()
    dims, box, cloud = _c4_cloud()
    w, h, c = dims
    up = torch.randn((h, w, c), generator=torch.Generator().manual_seed(5)).to(dev)
    plan = D.FvrPlan(cloud.n, dims, box.half, 0, dev)
    params = _params(cloud, dev)
    plan.bin(params)
    grads = torch.empty((5, cloud.n), dtype=torch.float64, device=dev)
    accum = torch.zeros(cloud.n, dtype=torch.float64, device=dev)
    plan.backward(params, up, grads, accum)
    g = grads.cpu().numpy()
    pick = np.random.default_rng(6).choice(cloud.n, 3000, replace=False)
    up_zyx = up.permute(2, 0, 1).contiguous().cpu().numpy()
    dm, ds, di, acc, _ = O.splat_bwd(cloud.mu[pick], cloud.sigma[pick], cloud.intensity[pick],
                                     box.shape, dims, up_zyx)
    assert rel_l2(g[0:3, pick].T, dm) < GRAD_TOL
    assert rel_l2(g[3, pick], ds) < GRAD_TOL
    assert rel_l2(g[4, pick], di) < GRAD_TOL
    assert rel_l2(accum.cpu().numpy()[pick], acc) < GRAD_TOL


@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_projector_full_size_dot_and_slices(cfg):
    dev = D.require_cuda()
    if cfg == "c2":
        w = h = c = 256
        geom = core.ScanGeometry.fan(50, 512, 1.6, 512.0, 512.0)
        ogeom = O.Geometry.fan(50, 512, 1.6, 512.0, 512.0)
    else:
        w = h = c = 512
        geom = core.ScanGeometry.fan(100, 1024, 1.6, 1024.0, 1024.0)
        ogeom = O.Geometry.fan(100, 1024, 1.6, 1024.0, 1024.0)
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    gen = torch.Generator().manual_seed(7)
    x = torch.rand((h, w, c), generator=gen).to(dev)
    # non-negative x and y: no cancellation in the f64 dot products, so the
    # 1e-5 bound measures the transpose, not f32 rounding of a near-zero sum
    y = torch.rand((geom.n_views, geom.n_detectors, c), generator=gen).to(dev)
    ax = op.forward(x)
    aty = op.adjoint(y)
    lhs = float((ax.double() * y.double()).sum())
    rhs = float((x.double() * aty.double()).sum())
    assert abs(lhs - rhs) / abs(lhs) < 1e-5
    for z in (0, c // 2 + 1, c - 1):
        xs = x[:, :, z].cpu().numpy()[None]                 # (1, h, w)
        assert rel_l2(ax[:, :, z:z + 1].cpu().numpy(), O.project_forward(xs, ogeom)) < VOL_TOL
        ys = y[:, :, z:z + 1].cpu().numpy()
        assert rel_l2(aty[:, :, z].cpu().numpy()[None],
                      O.project_adjoint(ys, ogeom, (w, h, 1))) < VOL_TOL
    del op, x, y, ax, aty
    torch.cuda.empty_cache()


def test_loss_full_c2_sinogram():
    rng = np.random.default_rng(8)
    m, n, p = 50, 512, 256
    ref = rng.uniform(0, 60, (m, n, p)).astype(np.float32)
    pred = (ref + rng.normal(0, 2.0, ref.shape)).astype(np.float32)
    vol = rng.uniform(0, 1, (32, 40, 48)).astype(np.float32)
    v, gp, gv, parts = loss.total_loss_detailed(core.Sinogram.from_views(pred),
                                                core.Sinogram.from_views(ref),
                                                core.VolumeGrid.from_zyx(vol), loss.LossWeights())
    ov, ogp, ogv, oparts = O.total_loss_detailed(pred.astype(np.float64), ref.astype(np.float64),
                                                 vol.astype(np.float64))
    assert abs(v - ov) <= 1e-9 * max(1.0, abs(ov))
    for k in ("l1", "ssim", "tv"):
        assert abs(parts[k] - oparts[k]) <= 1e-9 * max(1.0, abs(oparts[k])), k
    assert rel_l2(gp, ogp) < 1e-6
    assert rel_l2(gv, ogv) < 1e-6
