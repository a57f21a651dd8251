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


# backward kernel variants: the spatially ordered persistent kernel (default),
# and the per-Gaussian-warp kernel with TMA-fed rows or direct loads
BWD_VARIANTS = {"ts": {"SPLATCT_BWD_KERNEL": "ts"}, "ts2": {"SPLATCT_BWD_KERNEL": "ts2"},
                "sp": {"SPLATCT_BWD_KERNEL": "sp"},
                "warp_tma": {"SPLATCT_BWD_KERNEL": "warp"},
                "warp_direct": {"SPLATCT_BWD_KERNEL": "warp", "SPLATCT_BWD_NO_TMA": "1"}}


@pytest.mark.parametrize("dims", [(40, 36, 32), (6, 5, 8), (64, 48, 256)])
def test_backward_variants_agree(dims, monkeypatch):
    """The backward kernels (tile-staged default, ordered, per-Gaussian warp with
    TMA rows or direct loads; TMA boxes zero-filled at tiny volumes; the
    full-box paths at c = 256) sum the same terms in different orders: equal
    to fp32 rounding, and each run-to-run bitwise."""
    rng = np.random.default_rng(9)
    box = core.BoxConfig.for_dims(17, dims)
    n = 1500
    mu = np.stack([rng.uniform(-3, d + 3, n) for d in dims], 1)
    cloud = core.GaussianCloud(mu, rng.uniform(0.5, 2.5, n), rng.uniform(0, 1, n))
    up = core.VolumeGrid.from_zyx(rng.standard_normal(dims[::-1]).astype(np.float32))
    out = {}
    for name, env in BWD_VARIANTS.items():
        for k in ("SPLATCT_BWD_KERNEL", "SPLATCT_BWD_NO_TMA", "SPLATCT_NO_TMA"):
            monkeypatch.delenv(k, raising=False)
        for k, v in env.items():
            monkeypatch.setenv(k, v)
        out[name] = fvr.backward(cloud, box, dims, up)
        again = fvr.backward(cloud, box, dims, up)
        np.testing.assert_array_equal(out[name].d_mu, again.d_mu)
        np.testing.assert_array_equal(out[name].d_sigma, again.d_sigma)
    a = out["warp_tma"]
    dm, ds, di, acc, _ = O.splat_bwd(mu, cloud.sigma, cloud.intensity, box.shape, dims, up.zyx)
    assert rel_l2(a.d_mu, dm) < GRAD_TOL and rel_l2(a.d_sigma, ds) < GRAD_TOL
    assert rel_l2(a.d_intensity, di) < GRAD_TOL
    for b in (out["ts"], out["ts2"], out["sp"], out["warp_direct"]):
        for x, y in ((a.d_mu, b.d_mu), (a.d_sigma, b.d_sigma), (a.d_intensity, b.d_intensity),
                     (a.accum_pos_grad_norm, b.accum_pos_grad_norm)):
            assert rel_l2(x, y) < 1e-6
    # the two tile-staged kernels share the per-Gaussian arithmetic: bitwise
    np.testing.assert_array_equal(out["ts"].d_mu, out["ts2"].d_mu)
    np.testing.assert_array_equal(out["ts"].d_sigma, out["ts2"].d_sigma)
    np.testing.assert_array_equal(out["ts"].d_intensity, out["ts2"].d_intensity)


def test_backward_tile_staged_dense_split_entries(monkeypatch):
    """A dense cloud (~900 first-tile Gaussians per 16^3 tile) overflows the
    asynchronous tile-staged kernel's 1024-Gaussian queue entries, so units and
    single tiles are split across entries, each re-staging its slabs.  The
    gradients match the per-Gaussian warp kernel (1e-6) and the synchronous
    tile-staged kernel (bitwise), run to run bitwise.  (The dispatcher's own
    choice of this kernel for dense clouds is exercised at C4 by
    test_gpu_fullsize.py::test_fvr_backward_c4_sampled.)"""
    rng = np.random.default_rng(12)
    dims = (64, 64, 64)
    box = core.BoxConfig.cube(17)
    n = 60000
    mu = np.stack([rng.uniform(0, d, n) for d in dims], 1)
    cloud = core.GaussianCloud(mu, rng.uniform(0.5, 2.5, n), rng.uniform(0, 1, n))
    up = core.VolumeGrid.from_zyx(rng.standard_normal(dims[::-1]).astype(np.float32))
    out = {}
    for name in ("warp", "ts", "ts2"):
        monkeypatch.setenv("SPLATCT_BWD_KERNEL", name)
        out[name] = fvr.backward(cloud, box, dims, up)
        again = fvr.backward(cloud, box, dims, up)
        np.testing.assert_array_equal(out[name].d_mu, again.d_mu)
    a = out["warp"]
    for b in (out["ts2"],):
        for x, y in ((a.d_mu, b.d_mu), (a.d_sigma, b.d_sigma), (a.d_intensity, b.d_intensity),
                     (a.accum_pos_grad_norm, b.accum_pos_grad_norm)):
            assert rel_l2(x, y) < 1e-6
    np.testing.assert_array_equal(out["ts2"].d_mu, out["ts"].d_mu)
    np.testing.assert_array_equal(out["ts2"].d_sigma, out["ts"].d_sigma)
    np.testing.assert_array_equal(out["ts2"].d_intensity, out["ts"].d_intensity)


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
    monkeypatch.setenv("SPLATCT_BWD_KERNEL", "warp")   # the visit-order switch of that kernel
    for o in ("0", "1"):
        monkeypatch.setenv("SPLATCT_BWD_ORDER", o)
        out.append(fvr.backward(cloud, box, dims, up))
    a, b = out
    for x, y in ((a.d_mu, b.d_mu), (a.d_sigma, b.d_sigma), (a.d_intensity, b.d_intensity),
                 (a.accum_pos_grad_norm, b.accum_pos_grad_norm)):
        np.testing.assert_array_equal(x, y)


def _footprint_union(mu, half, dims):
    """Boolean zyx mask of every voxel inside some Gaussian's clipped footprint
    (the reference's floor(mu) +- half, _kernels.py:45-47,61-78)."""
    w, h, c = dims
    m = np.zeros((c, h, w), bool)
    f = np.floor(mu).astype(np.int64)
    hx, hy, hz = half
    for (x, y, z) in f:
        x0, x1 = max(x - hx, 0), min(x + hx + 1, w)
        y0, y1 = max(y - hy, 0), min(y + hy + 1, h)
        z0, z1 = max(z - hz, 0), min(z + hz + 1, c)
        if x0 < x1 and y0 < y1 and z0 < z1:
            m[z0:z1, y0:y1, x0:x1] = True
    return m


@pytest.mark.parametrize("side", [9, 13, 15, 17])
@pytest.mark.parametrize("variant", sorted(BWD_VARIANTS))
def test_backward_never_reads_outside_footprints(side, variant, monkeypatch):
    """Upstream is NaN everywhere outside the union of footprints (what the
    masked adjoint leaves unwritten): gradients stay finite and match the
    oracle, on the TMA row path (c % 4 == 0) and the direct-load path, with
    boxes narrower than the 17-column TMA box and Gaussians clipped at x = 0."""
    for k, v in BWD_VARIANTS[variant].items():
        monkeypatch.setenv(k, v)
    rng = np.random.default_rng(20 + side)
    dims = (64, 48, 36)
    box = core.BoxConfig.cube(side)
    n = 60                                     # 25-80 % of the voxels covered
    mu = np.stack([rng.uniform(-2, d + 2, n) for d in dims], 1)
    mu[:10, 0] = rng.uniform(-1.0, 2.0, 10)   # clipped at x = 0
    sig = rng.uniform(0.5, 2.5, n)
    inten = rng.uniform(0, 1, n)
    cloud = core.GaussianCloud(mu, sig, inten)
    up = rng.standard_normal(dims[::-1]).astype(np.float32)
    inside = _footprint_union(mu, box.half, dims)
    assert (~inside).any()
    poisoned = up.copy()
    poisoned[~inside] = np.nan
    gr = fvr.backward(cloud, box, dims, core.VolumeGrid.from_zyx(poisoned))
    clean = np.where(inside, up, 0).astype(np.float32)
    dm, ds, di, acc, _ = O.splat_bwd(mu, sig, inten, box.shape, dims, clean)
    for got, want in ((gr.d_mu, dm), (gr.d_sigma, ds), (gr.d_intensity, di),
                      (gr.accum_pos_grad_norm, acc)):
        assert np.all(np.isfinite(got))
        assert rel_l2(got, want) < GRAD_TOL


@pytest.mark.parametrize("side", [9, 13, 17])
def test_trainer_step_with_poisoned_adjoint_buffer(side):
    """A training step with the masked adjoint (<= 64 z tiles, c % 4 == 0) whose
    output buffer starts as NaN: the quads the adjoint skips stay NaN, and the
    voxelizer backward must never read them."""
    import torch
    from paper_2411_04844_b200 import device as D, loss
    from paper_2411_04844_b200.trainer import Trainer
    dev = D.require_cuda()
    dims = (48, 40, 32)
    box = core.BoxConfig.cube(side)
    rng = np.random.default_rng(30 + side)
    n = 150
    mu = np.stack([rng.uniform(-1, d / 2, n) for d in dims], 1)   # leaves empty space
    cloud = core.GaussianCloud(mu, rng.uniform(0.6, 1.5, n), rng.uniform(0, 1, n))
    geom = core.ScanGeometry.parallel(8, 64)
    meas = torch.rand((8, 64, dims[2]), device=dev)
    tr = Trainer(meas, geom, dims, box, loss.LossWeights(), D.cloud_to_params(cloud, dev),
                 max_iters=10, trace_cap=3)
    assert tr.fvr.footprint_coverage is not None   # the masked adjoint is on
    tr.dl.fill_(float("nan"))
    tr.initial_volume()
    for _ in range(3):
        tr.step()
    torch.cuda.synchronize()
    assert torch.isnan(tr.dl).any()                # skipped quads were left unwritten
    assert np.all(np.isfinite(tr.trace_rows()[:, 0]))
    assert torch.isfinite(tr.params).all() and torch.isfinite(tr.grads).all()


def test_pinned_output_pool_results_stay_valid():
    """run_reconstruction hands its volume out in a reusable page-locked array;
    results the caller keeps are never overwritten by later calls (the pool
    falls back to pageable arrays once two results are held)."""
    import gc
    from paper_2411_04844_b200 import device as D, optim, phantom, projector
    dims = (40, 36, 32)
    truth = phantom.shepp_logan_3d(*dims)
    geom = core.ScanGeometry.parallel(12, 48)
    meas = projector.forward_project(truth, geom)
    box = core.BoxConfig.for_dims(17, dims)
    st = optim.ReconstructionSettings(dims=dims, box=box, max_iters=3, n_gaussians=500,
                                      densify_interval=0)
    cl = optim.init_cloud_random(dims, 500, seed=1, box=box)
    vols = [optim.run_reconstruction(meas, geom, st, init_cloud=cl)[0] for _ in range(4)]
    ref = vols[0].zyx.copy()
    for v in vols:
        np.testing.assert_array_equal(v.zyx, ref)
    assert len({v.data.__array_interface__["data"][0] for v in vols}) == 4
    del vols
    gc.collect()
    assert all(not e.busy for e in D._OUT_POOL)
    v = optim.run_reconstruction(meas, geom, st, init_cloud=cl)[0]
    np.testing.assert_array_equal(v.zyx, ref)


@pytest.mark.parametrize("groups", ["band8", "band16"])
def test_projector_band_groups_match_4ray_groups(groups, monkeypatch):
    """The opt-in band forms of the forward operator (sliding 4-ray windows
    over 8 / 16-ray bands, SPLATCT_FWD_GROUPS) give the 4-ray-group forward
    to f32 summation order, densely and with empty-space skipping, and write
    every ray (the output starts as NaN; the fan is wider than the slice, so
    some rays touch no pixel).  Bands that cannot fit the build capacity are
    refused."""
    import torch
    from paper_2411_04844_b200 import device as D
    dev = D.require_cuda()
    w, h, c = 64, 48, 256
    geom = core.ScanGeometry.fan(24, 150, 1.1, 90.0, 70.0)
    g = torch.Generator(device="cpu").manual_seed(3)
    x = torch.randn((h, w, c), generator=g)
    x[:, :, 96:176] = 0.0                         # z tiles 6..10 all zero
    x[:20, :, :] = 0.0                            # and whole empty columns
    seg = (x.reshape(h, w, c // 16, 16) != 0).any(-1).numpy()    # (h, w, tiles)
    bits = (seg.astype(np.uint64) << np.arange(c // 16, dtype=np.uint64)).sum(-1, dtype=np.uint64)
    occ = torch.from_numpy(bits.reshape(-1).view(np.int64)).to(dev)
    x = x.to(dev)
    monkeypatch.setenv("SPLATCT_FWD_GROUPS", "4")
    ref = D.ProjectorOperator(geom, w, h, 0.5, dev)
    monkeypatch.setenv("SPLATCT_FWD_GROUPS", groups)
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    assert op.fkind == (3 if groups == "band8" else 4)
    a = ref.forward(x)
    for skip in (None, D.VP(occ.data_ptr())):
        b = torch.full_like(a, float("nan"))
        op.forward(x, out=b, occ=skip)
        assert torch.isfinite(b).all()
        assert rel_l2(b.cpu().numpy(), a.cpu().numpy()) < 1e-6
        again = op.forward(x, occ=skip)
        np.testing.assert_array_equal(again.cpu().numpy(), b.cpu().numpy())
    big = core.ScanGeometry.fan(8, 700, 1.6, 512.0, 512.0)
    monkeypatch.setenv("SPLATCT_FWD_GROUPS", "band16")
    with pytest.raises(ValueError):
        D.ProjectorOperator(big, 512, 512, 0.5, dev)


@pytest.mark.parametrize("geom,w,h", [
    (core.ScanGeometry.fan(50, 512, 1.6, 512.0, 512.0), 256, 256),
    (core.ScanGeometry.parallel(13, 70, 1.3), 41, 29),
    (core.ScanGeometry.fan(7, 20, 0.9, 12.0, 9.0), 5, 7)])
def test_march_segments_same_operator(geom, w, h, monkeypatch):
    """The operator's ray march split into segments per ray (a thread each)
    merges exactly the weights of the whole-ray march: every ray has the same
    (pixel, weight) entries bitwise, only their order inside the row differs,
    and the blocked operators built from them are identical."""
    import torch
    from paper_2411_04844_b200 import device as D
    dev = D.require_cuda()
    monkeypatch.setenv("SPLATCT_MARCH_SEGMENTS", "1")
    ref = D.ProjectorOperator(geom, w, h, 0.5, dev)
    monkeypatch.delenv("SPLATCT_MARCH_SEGMENTS")
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    assert torch.equal(ref.a_ptr, op.a_ptr) and ref.nnz == op.nnz > 0

    def rows_sorted(o):
        lens = o.a_ptr[1:] - o.a_ptr[:-1]
        row = torch.repeat_interleave(torch.arange(o.n_rays, device=dev), lens)
        perm = torch.argsort(row * (w * h) + o.a_col.long()[:o.nnz])
        return o.a_col[:o.nnz][perm], o.a_val[:o.nnz][perm]
    for u, v in zip(rows_sorted(ref), rows_sorted(op)):
        assert torch.equal(u, v)
    for x, y in ((ref.at_ptr, op.at_ptr), (ref.at_ray, op.at_ray), (ref.at_val, op.at_val)):
        assert torch.equal(x, y)
    for a, b in ((ref.fb, op.fb), (ref.ab, op.ab)):
        assert a[3] == b[3]
        for u, v in zip(a[:3], b[:3]):
            assert torch.equal(u, v)


@pytest.mark.parametrize("c", [256, 100, 1040])
def test_forward_cta_order_is_bitwise_neutral(c):
    """The blocked forward launched with its CTAs longest-first gives bitwise
    the default order's sinogram; the order covers every CTA once (c = 1040:
    a volume beyond ~3/4 of L2, z-chunk-major, ordered within each chunk)."""
    import ctypes
    import torch
    from paper_2411_04844_b200 import device as D
    from paper_2411_04844_b200._lib import call
    dev = D.require_cuda()
    w = h = 256 if c != 1040 else 176
    op = D.ProjectorOperator(core.ScanGeometry.fan(50, 512, 1.6, 512.0, 512.0), w, h, 0.5, dev)
    g = torch.Generator(device="cpu").manual_seed(11)
    vol = torch.rand((h, w, c), generator=g).to(dev)
    vol[:, :, : c // 3] = 0.0
    order = op._forward_order(c)
    ctas, zs, ordered = ctypes.c_int64(0), ctypes.c_int(0), ctypes.c_int(0)
    call("splatct_proj_forward_ctas", op.n_rays, op.fkind, w, h, c, ctypes.byref(ctas),
         ctypes.byref(zs), ctypes.byref(ordered))
    assert ordered.value == (2 if c == 1040 else 1)
    assert order is not None and order.numel() == ctas.value
    assert torch.equal(torch.sort(order.long()).values, torch.arange(ctas.value, device=dev))
    a = torch.full((op.m, op.n_det, c), float("nan"), device=dev)
    b = torch.full_like(a, float("nan"))
    fb = op.fb
    for dst, o in ((a, None), (b, order)):
        call("splatct_proj_forward_blocked_ordered", D.ptr(fb[0]), D.ptr(fb[1]), D.ptr(fb[2]),
             op.n_rays, op.fkind, D.ptr(vol), D.ptr(dst), c, D.VP(0), w, h, D.ptr(o), D.VP(0),
             D.stream_handle())
    assert torch.isfinite(a).all() and torch.equal(a, b)


def test_block_fill_needs_its_count_scratch():
    """The fill sizes its shared arrays from what the count left in the
    scratch: given a scratch its count did not fill, it fails loudly instead of
    building a wrong operator."""
    import ctypes
    import torch
    from paper_2411_04844_b200 import device as D
    from paper_2411_04844_b200._lib import SplatctError, call, size_query
    dev = D.require_cuda()
    op = D.ProjectorOperator(core.ScanGeometry.fan(50, 512, 1.6, 512.0, 512.0), 256, 256, 0.5,
                             dev)
    sb = size_query("splatct_proj_block_scratch_bytes", op.n_rays, 0, 256, 256)
    ng = (op.n_rays + 3) // 4
    gptr = torch.empty(ng + 1, dtype=torch.int64, device=dev)
    nb = ctypes.c_int64(0)
    dirs = op._group_dirs(4)
    scratch = torch.zeros(sb, dtype=torch.uint8, device=dev)
    call("splatct_proj_block_count", D.ptr(op.a_ptr), D.ptr(op.a_col), op.n_rays, 0, 256, 256,
         D.ptr(dirs), D.ptr(gptr), D.ptr(scratch), sb, ctypes.byref(nb), D.stream_handle())
    assert torch.equal(gptr, op.fb[0]) and nb.value == op.fb[3]
    gidx = torch.empty(nb.value, dtype=torch.int32, device=dev)
    gval = torch.empty((nb.value, 4), dtype=torch.float32, device=dev)
    fresh = torch.zeros(sb, dtype=torch.uint8, device=dev)
    with pytest.raises(SplatctError):
        call("splatct_proj_block_fill", D.ptr(op.a_ptr), D.ptr(op.a_col), D.ptr(op.a_val),
             op.n_rays, 0, 256, 256, D.ptr(dirs), D.ptr(gptr), D.ptr(gidx), D.ptr(gval),
             D.ptr(fresh), sb, D.stream_handle())
    call("splatct_proj_block_fill", D.ptr(op.a_ptr), D.ptr(op.a_col), D.ptr(op.a_val),
         op.n_rays, 0, 256, 256, D.ptr(dirs), D.ptr(gptr), D.ptr(gidx), D.ptr(gval),
         D.ptr(scratch), sb, D.stream_handle())
    assert torch.equal(gidx, op.fb[1]) and torch.equal(gval, op.fb[2])


@pytest.mark.parametrize("size", [256, 512, 37])
def test_block_build_without_sorts_matches_sort(size, monkeypatch):
    """The blocked operators built without sorting where the rows allow it --
    the count pass as a shared-memory hash set of the group's pixels, the
    pixel quads' fill as a merge of their ray-sorted rows -- are identical to
    the ones the bitonic sort builds (C2 / C4 fan geometries, a ragged one)."""
    import torch
    from paper_2411_04844_b200 import device as D
    dev = D.require_cuda()
    geom = {256: core.ScanGeometry.fan(50, 512, 1.6, 512.0, 512.0),
            512: core.ScanGeometry.fan(100, 1024, 1.6, 1024.0, 1024.0),
            37: core.ScanGeometry.parallel(11, 45, 1.2)}[size]
    monkeypatch.setenv("SPLATCT_BLOCK_COUNT", "sort")
    monkeypatch.setenv("SPLATCT_BLOCK_FILL", "sort")
    ref = D.ProjectorOperator(geom, size, size - size // 5, 0.5, dev)
    monkeypatch.delenv("SPLATCT_BLOCK_COUNT")
    monkeypatch.delenv("SPLATCT_BLOCK_FILL")
    op = D.ProjectorOperator(geom, size, size - size // 5, 0.5, dev)
    for a, b in ((ref.fb, op.fb), (ref.ab, op.ab)):
        assert a[3] == b[3]
        for u, v in zip(a[:3], b[:3]):
            assert torch.equal(u, v)


@pytest.mark.parametrize("dims,n", [((64, 48, 40), 3000), ((256, 256, 64), 20000)])
def test_row_ordered_bins_same_pairs(dims, n):
    """splatct_fvr_bin_row_ordered (the training step's bins): every tile holds
    the same (tile, Gaussian) pairs as the canonical bins, ordered by the
    footprint's first row relative to the tile (quantised), then by Gaussian;
    the forward over them matches the canonical forward to f32 rounding and is
    run-to-run bitwise (its k8-step skipping only drops exact zeros)."""
    import torch
    from paper_2411_04844_b200 import device as D, optim
    dev = D.require_cuda()
    box = core.BoxConfig.for_dims(17, dims)
    cloud = optim.init_cloud_random(dims, n, seed=5, box=box)
    params = D.cloud_to_params(cloud, dev)
    plan = D.FvrPlan(n, dims, box.half, 0, dev)
    plan.bin(params)
    fp, ts, items = plan.export_bins()
    vol_a = plan.forward(params, plan.new_volume()).cpu().numpy()
    plan.bin(params, row_ordered=True)
    fp2, ts2, items2 = plan.export_bins()
    vol_b = plan.forward(params, plan.new_volume()).cpu().numpy()
    vol_c = plan.forward(params, plan.new_volume()).cpu().numpy()
    np.testing.assert_array_equal(fp, fp2)
    np.testing.assert_array_equal(ts, ts2)
    nt = len(ts) - 1
    ty = (np.arange(nt) // ((dims[0] + 15) // 16)) % ((dims[1] + 15) // 16)
    tile_bits = int(np.ceil(np.log2(nt)))
    ybits = min(4, 8 * max(1, -(-tile_bits // 8)) - tile_bits)   # the radix key's spare bits
    reordered = 0
    for t in range(nt):
        a, b = items[ts[t]:ts[t + 1]], items2[ts[t]:ts[t + 1]]
        np.testing.assert_array_equal(np.sort(a), np.sort(b))
        np.testing.assert_array_equal(a, np.sort(a))          # canonical: ascending Gaussian
        # first footprint row relative to the tile, quantised; then ascending Gaussian
        q = np.clip(fp[b, 2] - 16 * ty[t] + 16, 0, 31) >> (5 - ybits)
        order = np.lexsort((b, q))
        np.testing.assert_array_equal(order, np.arange(len(b)))
        reordered += int(not np.array_equal(a, b))
    assert reordered > 0
    assert rel_l2(vol_b, vol_a) < 1e-6
    np.testing.assert_array_equal(vol_b, vol_c)


def test_adam_fused_into_bins_matches_separate_calls():
    """splatct_fvr_adam_bin (the training step's fused Adam + binning pass)
    leaves params and both moments bitwise as splatct_adam does, and bins the
    updated params exactly as a separate bin call would."""
    import torch
    from paper_2411_04844_b200 import device as D, optim
    dev = D.require_cuda()
    dims = (64, 48, 40)
    box = core.BoxConfig.for_dims(17, dims)
    cloud = optim.init_cloud_random(dims, 4000, seed=6, box=box)
    g = torch.Generator(device="cpu").manual_seed(6)
    p0 = D.cloud_to_params(cloud, dev)
    grads = (torch.randn(p0.shape, generator=g, dtype=torch.float64) * 0.05).to(dev)
    m1 = (torch.randn(p0.shape, generator=g, dtype=torch.float64) * 0.01).to(dev)
    m2 = (torch.rand(p0.shape, generator=g, dtype=torch.float64) * 0.01).to(dev)
    scal = torch.tensor([3e-2, 0.1, 0.001], dtype=torch.float64, device=dev)
    a = [t.clone() for t in (p0, m1, m2)]
    b = [t.clone() for t in (p0, m1, m2)]
    plan_a = D.FvrPlan(cloud.n, dims, box.half, 0, dev)
    plan_b = D.FvrPlan(cloud.n, dims, box.half, 0, dev)
    D.adam(a[0], grads, a[1], a[2], scal, 0.3, 8.0)
    plan_a.bin(a[0], row_ordered=True)
    plan_b.adam_bin(b[0], grads, b[1], b[2], scal, 0.3, 8.0, row_ordered=True)
    for x, y in zip(a, b):
        np.testing.assert_array_equal(x.cpu().numpy(), y.cpu().numpy())
    for x, y in zip(plan_a.export_bins(), plan_b.export_bins()):
        np.testing.assert_array_equal(x, y)
