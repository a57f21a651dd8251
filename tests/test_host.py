"""Host-side logic of the product package (no GPU needed)."""
import numpy as np
import pytest

from paper_2411_04844_b200 import core, densify, phantom, projector
from paper_2411_04844_b200.distributed import slab_bounds
from paper_2411_04844_b200.optim import OptimizerState, _holdout_split, init_cloud_random
from paper_2411_04844_b200.loss import LossWeights, ssim_valid_count


def test_offset_grid_and_box():
    assert core.make_offset_grid(core.BoxConfig(1, 1, 1)).offsets.tolist() == [[0, 0, 0]]
    assert core.make_offset_grid(core.BoxConfig(3, 1, 1)).offsets.tolist() == \
        [[-1, 0, 0], [0, 0, 0], [1, 0, 0]]
    g = core.make_offset_grid(core.BoxConfig.cube(17))
    assert len(g) == 4913 and g.offsets.min() == -8 and g.offsets.max() == 8
    assert (g.offsets.sum(axis=0) == 0).all()
    assert core.BoxConfig.for_dims(17, (64, 64, 1)).shape == (17, 17, 1)
    assert core.BoxConfig.for_dims(17, (10, 64, 4)).shape == (9, 17, 3)
    with pytest.raises(core.ValidationError):
        core.BoxConfig(2, 3, 3)


def test_cloud_validation_messages():
    assert core.validate_cloud(core.GaussianCloud([[0, 0, 0]], [1.0], [0.5])) == []
    msgs = core.validate_cloud(core.GaussianCloud([[0, 0, 0]], [-1.0], [0.5]))
    assert any("index 0, field sigma" in m for m in msgs)
    msgs = core.validate_cloud(core.GaussianCloud([[0, 0, 0], [1, 1, 1]], [1.0], [1.0, 1.0]))
    assert any("length mismatch" in m for m in msgs)
    with pytest.raises(core.ValidationError):
        core.require_valid_cloud(core.GaussianCloud(np.zeros((0, 3)), [], []))


def test_linear_index_bijection():
    dims = (3, 4, 5)
    idx = {core.linear_index(x, y, z, dims) for z in range(5) for y in range(4) for x in range(3)}
    assert idx == set(range(60))


def test_geometry_validation():
    core.ScanGeometry.parallel(25, 96)
    with pytest.raises(core.ValidationError):
        core.ScanGeometry("cone", 1, 1, 1.0, [0.0])
    g = core.ScanGeometry.fan(10, 20, 1.0, 10.0, 10.0)
    with pytest.raises(core.ValidationError):
        g.check_volume((64, 64, 1))
    with pytest.raises(core.ValidationError):
        core.Sinogram.from_views(np.full((2, 2, 1), np.nan))


def test_phantom_matches_reference(traj_golden):
    """Shepp-Logan 64^3 equals the reference's rasterisation bit for bit."""
    v = phantom.shepp_logan_3d(64, 64, 64)
    np.testing.assert_array_equal(v.zyx, traj_golden["traj_truth"])
    ch = phantom.chest_3d(64, 64, 64).zyx
    assert ch.min() >= 0.0 and ch.max() <= 1.0 and ch.max() > 0.5


def test_fbp_filter_kernel_equals_fft_filter():
    """Direct-convolution taps reproduce the zero-padded FFT ramp filter (projector.py:134-141)."""
    rng = np.random.default_rng(0)
    for n, sp, win in ((30, 1.0, "ramp"), (47, 0.8, "hann"), (96, 1.6, "ramp")):
        rows = rng.standard_normal((3, n))
        n_pad = int(2 ** np.ceil(np.log2(max(64, 2 * n))))
        resp = projector._ramp_response(n_pad, sp, win)
        ref = np.real(np.fft.ifft(np.fft.fft(rows, n=n_pad, axis=1) * resp, axis=1))[:, :n] * sp
        k = projector._filter_kernel(n, sp, win)
        out = np.array([[sum(k[i - j + n - 1] * r[j] for j in range(n)) for i in range(n)]
                        for r in rows])
        np.testing.assert_allclose(out, ref, rtol=1e-10, atol=1e-12)


def test_densify_spec_examples():
    """SPEC.md densify examples (clone halves intensity, split divides sigma by cbrt 2, prune)."""
    p = densify.DensifyParams(tau=2e-4, theta=1.0, box_size=17, grad_prune_enabled=True)
    rng = np.random.default_rng(0)

    def grads(avg):
        n = len(avg)
        return core.ParamGradients(np.zeros((n, 3)), np.zeros(n), np.zeros(n), np.asarray(avg), 1)

    c = core.GaussianCloud([[5, 5, 5]], [0.5], [0.8])
    new, rep = densify.densify_and_prune(c, grads([1e-3]), p, rng)
    assert rep.clones == 1 and new.n == 2 and np.all(new.intensity == 0.4)
    c = core.GaussianCloud([[5, 5, 5]], [2.0], [0.8])
    new, rep = densify.densify_and_prune(c, grads([1e-3]), p, rng)
    assert rep.splits == 1 and new.n == 2 and np.allclose(new.sigma, 2.0 / np.cbrt(2.0))
    c = core.GaussianCloud([[5, 5, 5]], [3.5 * 17], [0.8])
    new, rep = densify.densify_and_prune(c, grads([1e-3]), p, rng)
    assert rep.prunes == 1 and new.n == 0
    c = core.GaussianCloud([[5, 5, 5]] * 3, [0.5] * 3, [0.8] * 3)
    new, rep = densify.densify_and_prune(c, grads([1e-3] * 3), densify.DensifyParams(n_max=3), rng)
    assert new.n == 3 and rep.clones == 0


def test_slab_bounds_cover():
    for c, world in ((64, 2), (512, 8), (257, 4), (5, 8)):
        slabs = [slab_bounds(c, world, r) for r in range(world)]
        z = 0
        for s in slabs:
            assert s.z0 == z and s.c_global == c
            z += s.c_local
        assert z == c


def test_lr_schedule_and_state():
    st = OptimizerState.fresh(4, 3e-4, 3e-5, 500)
    assert st.lr() == 3e-4
    from dataclasses import replace
    assert abs(replace(st, step=500).lr() - 3e-5) < 1e-18
    assert abs(replace(st, step=900).lr() - 3e-5) < 1e-18


def test_misc_helpers():
    assert ssim_valid_count(25, 96) == 15 * 86
    assert ssim_valid_count(5, 40) == 1 * 30
    with pytest.raises(core.ValidationError):
        LossWeights(0, 0, 0)
    cl = init_cloud_random((64, 64, 64), 100, seed=0)
    assert cl.mu.min() >= 8 and cl.mu.max() <= 56
    g = core.ScanGeometry.parallel(20, 8)
    s = core.Sinogram.from_views(np.zeros((20, 8, 1)))
    (gt, st), (gv, sv) = _holdout_split(g, s, 0.1)
    assert gt.n_views + gv.n_views == 20 and gv.n_views == 2


def test_densify_matches_reference_golden():
    """Host restatement == the reference's densify_and_prune + remap, bitwise."""
    from densify_golden import cases
    from paper_2411_04844_b200 import optim
    for ci, cloud, grads, prm, (seed, it), g in cases():
        new, rep = densify.densify_and_prune(cloud, grads, prm, np.random.default_rng([seed, it]))
        assert [rep.clones, rep.splits, rep.prunes, rep.n_after] == g["report"].tolist(), ci
        np.testing.assert_array_equal(rep.kept, g["kept"])
        np.testing.assert_array_equal(new.mu, g["out_mu"])
        np.testing.assert_array_equal(new.sigma, g["out_sigma"])
        np.testing.assert_array_equal(new.intensity, g["out_intensity"])
        n = cloud.n
        st = optim.OptimizerState(g["in_m_mu"], g["in_v_mu"], g["in_m_sigma"], g["in_v_sigma"],
                                  g["in_m_intensity"], g["in_v_intensity"], 5, 3e-4, 3e-5, 100)
        assert st.n == n
        st2 = st.remap(rep)
        for k in ("m_mu", "v_mu", "m_sigma", "v_sigma", "m_intensity", "v_intensity"):
            np.testing.assert_array_equal(getattr(st2, k), g["out_" + k])
