"""The CPU oracle (oracle/) is pinned against vectors produced by the real
reference (tests/golden/make_golden.py).  CPU only."""
import numpy as np
import pytest

from conftest import rel_l2
from oracle import oracle as O


def _geom(g, ci):
    p = lambda k: g[f"proj{ci}_{k}"]
    return O.Geometry(str(p("variant")) == "fan", p("angles"), int(p("n_det")),
                      float(p("spacing")), float(p("rs")), float(p("rd")))


def test_fvr_forward_backward(kernels_golden):
    g = kernels_golden
    for ci in range(int(g["fvr_ncases"])):
        p = lambda k: g[f"fvr{ci}_{k}"]
        dims, box = tuple(p("dims")), tuple(p("box"))
        vol = O.splat_fwd(p("mu"), p("sigma"), p("intensity"), box, dims)
        np.testing.assert_array_equal(vol, p("vol"))
        dm, ds, di, acc, it = O.splat_bwd(p("mu"), p("sigma"), p("intensity"), box, dims, p("up"))
        assert rel_l2(dm, p("d_mu")) < 1e-13
        assert rel_l2(ds, p("d_sigma")) < 1e-13
        assert rel_l2(di, p("d_intensity")) < 1e-13
        assert rel_l2(acc, p("accum")) < 1e-13 and it == 1


def test_spec_known_answers(kernels_golden):
    """SPEC.md:134-135 single-Gaussian values."""
    v = O.splat_fwd([[8.0, 8, 8]], [1.0], [1.0], (17, 17, 17), (17, 17, 17))
    assert v[8, 8, 8] == np.float32(1.0)
    assert abs(v[8, 8, 9] - np.exp(-0.5)) < 1e-7
    np.testing.assert_array_equal(v, kernels_golden["spec_v_int"])
    v2 = O.splat_fwd([[8.5, 8, 8]], [1.0], [1.0], (17, 17, 17), (17, 17, 17))
    np.testing.assert_array_equal(v2, kernels_golden["spec_v_half"])
    assert abs(v2[8, 8, 8] - np.exp(-0.125)) < 1e-7 and v2[8, 8, 8] == v2[8, 8, 9]


def test_nodecomp_and_direct_agree():
    rng = np.random.default_rng(3)
    mu = rng.uniform(8, 24, (20, 3))
    sg = rng.uniform(0.5, 1.5, 20)
    it = rng.uniform(0, 1, 20)
    a = O.splat_fwd(mu, sg, it, (17, 17, 17), (32, 32, 32))
    b = O.splat_plain(mu, sg, it, (17, 17, 17), (32, 32, 32))
    c = O.splat_direct(mu, sg, it, (32, 32, 32))
    assert np.abs(a - b).max() <= 1e-5
    assert np.abs(a - c).max() <= 1e-4 * np.abs(c).max()


def test_projector(kernels_golden):
    g = kernels_golden
    for ci in range(int(g["proj_ncases"])):
        p = lambda k: g[f"proj{ci}_{k}"]
        geom = _geom(g, ci)
        np.testing.assert_array_equal(O.project_forward(p("vol"), geom), p("sino"))
        np.testing.assert_array_equal(O.project_adjoint(p("ys"), geom, tuple(p("dims"))), p("bp"))


def test_loss(kernels_golden):
    g = kernels_golden
    for ci in range(int(g["loss_ncases"])):
        p = lambda k: g[f"loss{ci}_{k}"]
        v, gp, gv, parts = O.total_loss_detailed(p("pred"), p("ref"), p("vol"))
        assert abs(v - float(p("total"))) < 1e-12
        assert abs(parts["l1"] - float(p("l1"))) < 1e-14
        assert abs(parts["ssim"] - float(p("ssim"))) < 1e-12
        assert abs(parts["tv"] - float(p("tv"))) < 1e-14
        assert rel_l2(gp, p("grad_pred")) < 1e-12
        np.testing.assert_array_equal(gv, p("grad_vol"))


def test_adam(kernels_golden):
    g = kernels_golden
    st = dict(step=int(g["adam_step"]), lr0=3e-4, lrf=3e-5, max_iters=100)
    for k in ("m_mu", "v_mu", "m_sigma", "v_sigma", "m_intensity", "v_intensity"):
        st[k] = g[f"adam_in_{k}"]
    mu, s, i, st2 = O.adam_step(g["adam_in_mu"], g["adam_in_sigma"], g["adam_in_intensity"],
                                g["adam_d_mu"], g["adam_d_sigma"], g["adam_d_intensity"], st, 51.0)
    np.testing.assert_array_equal(mu, g["adam_out_mu"])
    np.testing.assert_array_equal(s, g["adam_out_sigma"])
    np.testing.assert_array_equal(i, g["adam_out_intensity"])
    for k in ("m_mu", "v_mu", "m_sigma", "v_sigma", "m_intensity", "v_intensity"):
        np.testing.assert_array_equal(st2[k], g[f"adam_out_{k}"])


def test_trajectory_prefix(traj_golden):
    """First 6 iterations of the config-1 run (max_iters=500) match the reference."""
    g = traj_golden
    geom = O.Geometry.parallel(25, 96)
    _, _, tr = O.train(g["traj_meas"], geom, (64, 64, 64), (17, 17, 17), g["traj_init_mu"],
                       g["traj_init_sigma"], g["traj_init_intensity"], 500, iters_to_run=6,
                       truth=g["traj_truth"])
    for r in tr:
        k = r["iteration"] - 1
        assert abs(r["loss"] - g["traj_loss"][k]) < 1e-12
        assert abs(r["psnr"] - g["traj_psnr"][k]) < 1e-9


def test_bins_restatement():
    """Footprints clip to the volume with a true floor; lists ascending per tile."""
    mu = np.array([[-0.5, 3.25, 2.0], [8.0, 8.0, 8.0], [31.9, 40.0, 5.0], [15.99, 16.0, 0.0]])
    fp, ts, items = O.bins(mu, (17, 17, 17), (32, 32, 32), (16, 16, 16))
    assert list(fp[0]) == [0, 7, 0, 11, 0, 10]          # floor(-0.5) = -1
    assert list(fp[2][2:4]) == [1, 0]                      # y footprint empty (40-8 > 31)
    assert ts[-1] == len(items)
    for t in range(len(ts) - 1):
        seg = items[ts[t]:ts[t + 1]]
        assert np.all(np.diff(seg) > 0)
    assert 2 not in items
