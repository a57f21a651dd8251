"""Device densification (csrc/densify.cu) against the reference's own
densify_and_prune + OptimizerState.remap outputs (tests/golden/densify.npz),
bitwise: masks, top-k budgets, compaction order, clone halving, split
children mu + N(0,1) sigma and sigma / cbrt 2, carried / zeroed moments."""
import numpy as np
import pytest
import torch

from densify_golden import cases

pytestmark = pytest.mark.gpu

from paper_2411_04844_b200 import core, densify, device as D, optim  # noqa: E402


def _moments(g, pre):
    m = np.empty((5, g[pre + "m_mu"].shape[0]))
    v = np.empty_like(m)
    m[0:3], m[3], m[4] = g[pre + "m_mu"].T, g[pre + "m_sigma"], g[pre + "m_intensity"]
    v[0:3], v[3], v[4] = g[pre + "v_mu"].T, g[pre + "v_sigma"], g[pre + "v_intensity"]
    return m, v


@pytest.mark.parametrize("case", range(5))
def test_device_densify_matches_reference(case):
    dev = D.require_cuda()
    ci, cloud, grads, prm, (seed, it), g = cases()[case]
    m_in, v_in = _moments(g, "in_")
    params = D.cloud_to_params(cloud, dev)
    accum = torch.from_numpy(grads.accum_pos_grad_norm.copy()).to(dev)
    p2, m1, m2, rep = D.densify(params, torch.from_numpy(m_in).to(dev),
                                torch.from_numpy(v_in).to(dev), accum, grads.iters_since_densify,
                                prm, np.random.default_rng([seed, it]))
    assert [rep.clones, rep.splits, rep.prunes, rep.n_after] == g["report"].tolist()
    out = D.params_to_cloud(p2)
    np.testing.assert_array_equal(out.mu, g["out_mu"])
    np.testing.assert_array_equal(out.sigma, g["out_sigma"])
    np.testing.assert_array_equal(out.intensity, g["out_intensity"])
    m_out, v_out = _moments(g, "out_")
    np.testing.assert_array_equal(m1.cpu().numpy(), m_out)
    np.testing.assert_array_equal(m2.cpu().numpy(), v_out)


@pytest.mark.parametrize("n,k_off", [(20000, 1), (20000, 3000), (200000, 12345)])
def test_device_topk_budget_large(n, k_off):
    """Radix-select top-k at larger sizes (clone budget binds) == host restatement."""
    dev = D.require_cuda()
    rng = np.random.default_rng(n + k_off)
    mu = rng.uniform(0, 64, (n, 3))
    sigma = rng.uniform(0.3, 0.9, n)              # all clone candidates when hot
    inten = rng.uniform(0, 1, n)
    accum = rng.uniform(1e-4, 1e-2, n) * 10
    cloud = core.GaussianCloud(mu, sigma, inten)
    prm = densify.DensifyParams(n_max=n + k_off, tau=2e-4, theta=1.0)
    g = core.ParamGradients(np.zeros((n, 3)), np.zeros(n), np.zeros(n), accum, 10)
    new, rep = densify.densify_and_prune(cloud, g, prm, np.random.default_rng(0))
    z = torch.zeros((5, n), dtype=torch.float64, device=dev)
    p2, _, _, drep = D.densify(D.cloud_to_params(cloud, dev), z, z.clone(),
                               torch.from_numpy(accum).to(dev), 10, prm,
                               np.random.default_rng(0))
    assert (drep.clones, drep.splits, drep.prunes, drep.n_after) == \
        (rep.clones, rep.splits, rep.prunes, rep.n_after)
    out = D.params_to_cloud(p2)
    np.testing.assert_array_equal(out.mu, new.mu)
    np.testing.assert_array_equal(out.intensity, new.intensity)


def test_device_topk_ties_lowest_index_first():
    """Equal scores at the cut: the set is the k best, ties taken by lower index."""
    dev = D.require_cuda()
    n = 1000
    accum = np.full(n, 5e-3)
    accum[::7] = 9e-3                     # 143 strictly better ones
    cloud = core.GaussianCloud(np.full((n, 3), 10.0), np.full(n, 0.5), np.ones(n))
    k = 200
    prm = densify.DensifyParams(n_max=n + k, tau=2e-4, theta=1.0)
    z = torch.zeros((5, n), dtype=torch.float64, device=dev)
    p2, _, _, rep = D.densify(D.cloud_to_params(cloud, dev), z, z.clone(),
                              torch.from_numpy(accum).to(dev), 1, prm, np.random.default_rng(0))
    assert rep.clones == k and rep.n_after == n + k
    inten = D.params_to_cloud(p2).intensity[:n]        # originals, in index order
    halved = np.flatnonzero(inten == 0.5)
    best = np.flatnonzero(accum == 9e-3)
    ties = np.setdiff1d(np.arange(n), best)[:k - best.size]
    np.testing.assert_array_equal(halved, np.union1d(best, ties))


def test_run_reconstruction_device_densify_event():
    """An event inside run_reconstruction: trace counts == the host restatement
    applied to the same pre-event state."""
    from paper_2411_04844_b200 import phantom, projector
    dims = (32, 32, 32)
    truth = phantom.shepp_logan_3d(*dims)
    geom = core.ScanGeometry.parallel(12, 48)
    meas = projector.forward_project(truth, geom)
    box = core.BoxConfig.for_dims(17, dims)
    prm = densify.DensifyParams(grad_prune_enabled=False, tau=1e-9, theta=1.0, n_max=1300)
    kw = dict(dims=dims, box=box, n_gaussians=800, init_mode="fbp", seed=3, densify=prm)
    # pre-event state after 3 iterations (densify off), then one host event
    st3 = optim.ReconstructionSettings(max_iters=3, densify_interval=0, **kw)
    _, cl3, _ = optim.run_reconstruction(meas, geom, st3)
    st = optim.ReconstructionSettings(max_iters=5, densify_interval=3, **kw)
    _, cl, trace = optim.run_reconstruction(meas, geom, st)
    ev = trace[2]
    assert ev.clones + ev.splits > 0 and ev.n_gaussians == trace[3].n_gaussians
    assert ev.n_gaussians == 800 + ev.clones + ev.splits - ev.prunes <= 1300
    assert cl.n == ev.n_gaussians and np.all(np.isfinite(cl.mu))
    assert cl3.n == 800
