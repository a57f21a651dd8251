"""Edge cases of the voxelizer and projector against the CPU oracle.

Centres outside the volume (negative coordinates: true floor), boxes clipped
by the volume, per-axis box clamping on tiny / flat dims, dims that are not
multiples of the 16^3 tile or of 4 slices (scalar store paths), boxes larger
than 17 (the general backward path), an empty cloud, and the projector on
ragged slab depths.  Tolerances as in test_gpu_parity.py.
"""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import oracle as O

pytestmark = [pytest.mark.gpu,
              pytest.mark.filterwarnings("ignore:Gaussian centers outside the volume")]

from paper_2411_04844_b200 import core, fvr, projector  # noqa: E402

VOL_TOL = 1e-5
GRAD_TOL = 1e-4


def _check(mu, sig, inten, box, dims, seed=0):
    cloud = core.GaussianCloud(mu, sig, inten)
    vol = fvr.reconstruct(cloud, box, dims)
    ovol = O.splat_fwd(mu, sig, inten, box.shape, dims)
    if np.abs(ovol).max() == 0:
        assert np.abs(vol.zyx).max() == 0
    else:
        assert rel_l2(vol.zyx, ovol) < VOL_TOL
    up = np.random.default_rng(seed).standard_normal(dims[::-1]).astype(np.float32)
    gr = fvr.backward(cloud, box, dims, core.VolumeGrid.from_zyx(up))
    dm, ds, di, acc, _ = O.splat_bwd(mu, sig, inten, box.shape, dims, up)
    for got, want in ((gr.d_mu, dm), (gr.d_sigma, ds), (gr.d_intensity, di),
                      (gr.accum_pos_grad_norm, acc)):
        if np.abs(want).max() == 0:
            assert np.abs(got).max() == 0
        else:
            assert rel_l2(got, want) < GRAD_TOL


def test_centres_outside_and_clipped_boxes():
    """Centres up to a box beyond every face (incl. negative: floor, not trunc)."""
    rng = np.random.default_rng(1)
    dims = (40, 36, 33)
    box = core.BoxConfig.cube(17)
    n = 3000
    lo = -12.0
    mu = np.stack([rng.uniform(lo, d + 12.0, n) for d in dims], 1)
    mu[:20, 0] = rng.uniform(-9.5, -8.5, 20)     # boxes just touching / missing x = 0
    mu[20:40, 2] = rng.uniform(dims[2] + 7.5, dims[2] + 8.5, 20)
    _check(mu, rng.uniform(0.5, 3.0, n), rng.uniform(0, 1, n), box, dims)


@pytest.mark.parametrize("dims", [(20, 9, 5), (37, 23, 19), (16, 16, 1), (3, 50, 7),
                                  (6, 5, 8), (9, 20, 4)])
def test_flat_and_ragged_dims(dims):
    """Per-axis box clamping (BoxConfig.for_dims) and non-tile-multiple dims."""
    rng = np.random.default_rng(2)
    box = core.BoxConfig.for_dims(17, dims)
    n = 800
    mu = np.stack([rng.uniform(-2, d + 2, n) for d in dims], 1)
    _check(mu, rng.uniform(0.4, 2.5, n), rng.uniform(0, 1, n), box, dims)


def test_large_box_general_paths():
    """A 25^3 box: more tiles per Gaussian and the general backward path."""
    rng = np.random.default_rng(3)
    dims = (64, 48, 40)
    box = core.BoxConfig.cube(25)
    n = 1500
    mu = np.stack([rng.uniform(0, d, n) for d in dims], 1)
    _check(mu, rng.uniform(1.0, 4.0, n), rng.uniform(0, 1, n), box, dims)


def test_anisotropic_box():
    rng = np.random.default_rng(4)
    dims = (48, 40, 36)
    box = core.BoxConfig(9, 17, 5)
    n = 1200
    mu = np.stack([rng.uniform(0, d, n) for d in dims], 1)
    _check(mu, rng.uniform(0.5, 2.0, n), rng.uniform(0, 1, n), box, dims)


def test_empty_cloud_is_rejected():
    with pytest.raises(core.ValidationError):
        fvr.reconstruct(core.GaussianCloud(np.zeros((0, 3)), [], []), core.BoxConfig.cube(17),
                        (16, 16, 16))


@pytest.mark.parametrize("c", [1, 3, 37, 130])
def test_projector_ragged_depths(c):
    """Slab depths that select the scalar / float2 / float4 z-vector paths."""
    rng = np.random.default_rng(5)
    w, h = 30, 26
    zyx = rng.uniform(0, 1, (c, h, w)).astype(np.float32)
    geom = core.ScanGeometry.fan(9, 40, 1.1, 60.0, 40.0)
    sino = projector.forward_project(core.VolumeGrid.from_zyx(zyx), geom)
    osino = O.project_forward(zyx, O.Geometry.fan(9, 40, 1.1, 60.0, 40.0), 0.5)
    assert rel_l2(sino.views, osino) < VOL_TOL
    g = rng.standard_normal(sino.views.shape).astype(np.float32)
    bp = projector.back_project(core.Sinogram.from_views(g), geom, (w, h, c))
    obp = O.project_adjoint(g, O.Geometry.fan(9, 40, 1.1, 60.0, 40.0), (w, h, c), 0.5)
    assert rel_l2(bp.zyx, obp) < VOL_TOL


def test_deep_volume_has_no_occupancy_mask():
    """More than 64 z tiles: no occupancy words (the step stays dense) and the
    training step still runs through the same stages."""
    import torch
    from paper_2411_04844_b200 import device as D, loss
    from paper_2411_04844_b200.trainer import Trainer
    dev = D.require_cuda()
    dims = (24, 20, 1040)
    box = core.BoxConfig.cube(9)
    plan = D.FvrPlan(10, dims, box.half, 0, dev)
    assert plan.pixel_occupancy is None and plan.footprint_coverage is None
    assert plan.pixel_occupancy_words() is None
    rng = np.random.default_rng(7)
    n = 200
    mu = np.stack([rng.uniform(2, d - 2, n) for d in dims], 1)
    cloud = core.GaussianCloud(mu, rng.uniform(0.6, 1.5, n), rng.uniform(0, 1, n))
    geom = core.ScanGeometry.parallel(6, 30)
    meas = torch.rand((6, 30, dims[2]), device=dev)
    tr = Trainer(meas, geom, dims, box, loss.LossWeights(), D.cloud_to_params(cloud, dev),
                 max_iters=10, trace_cap=2)
    tr.initial_volume()
    tr.step()
    tr.step()
    assert np.all(np.isfinite(tr.trace_rows()[:, 0]))


@pytest.mark.parametrize("dims", [(40, 36, 32), (6, 5, 8)])
def test_backward_tma_rows_match_direct_loads(dims, monkeypatch):
    """The TMA-fed backward (c % 4 == 0; boxes larger than tiny volumes are
    zero-filled by the tensor map) against the direct-load path, which sums the
    same terms in another column order."""
    rng = np.random.default_rng(9)
    box = core.BoxConfig.for_dims(17, dims)
    n = 1500
    mu = np.stack([rng.uniform(-3, d + 3, n) for d in dims], 1)
    cloud = core.GaussianCloud(mu, rng.uniform(0.5, 2.5, n), rng.uniform(0, 1, n))
    up = core.VolumeGrid.from_zyx(rng.standard_normal(dims[::-1]).astype(np.float32))
    a = fvr.backward(cloud, box, dims, up)
    monkeypatch.setenv("SPLATCT_BWD_NO_TMA", "1")
    b = fvr.backward(cloud, box, dims, up)
    for x, y in ((a.d_mu, b.d_mu), (a.d_sigma, b.d_sigma), (a.d_intensity, b.d_intensity),
                 (a.accum_pos_grad_norm, b.accum_pos_grad_norm)):
        assert rel_l2(x, y) < 1e-6


@pytest.mark.parametrize("dims", [(40, 36, 32), (6, 5, 8)])
def test_forward_tma_store_matches_vector_stores(dims, monkeypatch):
    """The TMA bulk tensor store and the vector-store path write the same
    accumulators: bitwise-equal volumes (tiles clipped at the edges)."""
    rng = np.random.default_rng(10)
    box = core.BoxConfig.for_dims(17, dims)
    n = 1500
    mu = np.stack([rng.uniform(-3, d + 3, n) for d in dims], 1)
    cloud = core.GaussianCloud(mu, rng.uniform(0.5, 2.5, n), rng.uniform(0, 1, n))
    a = fvr.reconstruct(cloud, box, dims).zyx
    monkeypatch.setenv("SPLATCT_NO_TMA", "1")
    b = fvr.reconstruct(cloud, box, dims).zyx
    np.testing.assert_array_equal(a, b)


def test_backward_visit_order_is_bitwise_neutral(monkeypatch):
    """Index order and tile order only change which warp takes a Gaussian;
    each Gaussian's sums run in one warp in fixed order."""
    rng = np.random.default_rng(11)
    dims = (48, 40, 36)
    box = core.BoxConfig.cube(17)
    n = 2000
    mu = np.stack([rng.uniform(0, d, n) for d in dims], 1)
    cloud = core.GaussianCloud(mu, rng.uniform(0.5, 2.5, n), rng.uniform(0, 1, n))
    up = core.VolumeGrid.from_zyx(rng.standard_normal(dims[::-1]).astype(np.float32))
    out = []
    for o in ("0", "1"):
        monkeypatch.setenv("SPLATCT_BWD_ORDER", o)
        out.append(fvr.backward(cloud, box, dims, up))
    a, b = out
    for x, y in ((a.d_mu, b.d_mu), (a.d_sigma, b.d_sigma), (a.d_intensity, b.d_intensity),
                 (a.accum_pos_grad_norm, b.accum_pos_grad_norm)):
        np.testing.assert_array_equal(x, y)
