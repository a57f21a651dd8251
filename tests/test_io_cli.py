"""Raw + sidecar formats and the CLI.

CPU tests cover bit-exact round trips, config validation and the host-only
commands; the GPU test drives phantom -> project -> reconstruct -> metrics.
"""
import json
import os

import numpy as np
import pytest

from paper_2411_04844_b200 import cli, core, io as fio, phantom


def test_volume_round_trip_bit_exact(tmp_path):
    rng = np.random.default_rng(0)
    zyx = rng.standard_normal((5, 7, 9)).astype(np.float32)
    vol = core.VolumeGrid.from_zyx(zyx)
    p = str(tmp_path / "v.raw")
    fio.write_volume(p, vol)
    back = fio.read_volume(p)
    assert back.dims == (9, 7, 5)
    assert back.zyx.tobytes() == vol.zyx.tobytes()
    meta = json.load(open(p + ".json"))
    assert meta["kind"] == "volume" and meta["dims"] == [9, 7, 5]
    assert meta["min"] == float(zyx.min()) and meta["max"] == float(zyx.max())
    # idx order: x fastest (core.py:58-95)
    raw = np.fromfile(p, dtype="<f4")
    assert raw[core.linear_index(3, 2, 1, vol.dims)] == vol.at(3, 2, 1)


def test_sinogram_and_geometry_round_trip(tmp_path):
    geom = core.ScanGeometry.fan(12, 20, 1.3, 80.0, 60.0, 0.1, np.pi / 2)
    sino = core.Sinogram.from_views(np.arange(12 * 20 * 3, dtype=np.float32).reshape(12, 20, 3))
    p = str(tmp_path / "s.raw")
    fio.write_sinogram(p, sino, geom)
    back, g = fio.read_sinogram(p)
    assert back.views.tobytes() == sino.views.tobytes()
    assert g.key() == geom.key()


def test_cloud_round_trip(tmp_path):
    rng = np.random.default_rng(1)
    cl = core.GaussianCloud(rng.uniform(0, 30, (11, 3)), rng.uniform(0.5, 2, 11),
                            rng.uniform(0, 1, 11))
    p = str(tmp_path / "c.raw")
    fio.write_cloud(p, cl, {"iterations": 3})
    back = fio.read_cloud(p)
    assert back.mu.tobytes() == np.asarray(cl.mu, np.float64).tobytes()
    assert back.sigma.tobytes() == np.asarray(cl.sigma, np.float64).tobytes()
    assert back.intensity.tobytes() == np.asarray(cl.intensity, np.float64).tobytes()


def test_reader_rejects_bad_files(tmp_path):
    p = str(tmp_path / "v.raw")
    with pytest.raises(core.ValidationError):
        fio.read_volume(p)
    fio.write_volume(p, core.VolumeGrid.zeros((4, 4, 4)))
    with pytest.raises(core.ValidationError):
        fio.read_sinogram(p)                     # wrong kind
    np.zeros(10, "<f4").tofile(p)
    with pytest.raises(core.ValidationError):
        fio.read_volume(p)                       # size mismatch


def test_geometry_from_dict_limited_angle():
    g = fio.geometry_from_dict({"variant": "parallel", "n_views": 8, "n_detectors": 16,
                                "angle_start": 0.0, "angle_extent": np.pi / 2})
    assert g.view_angles.max() < np.pi / 2
    with pytest.raises(core.ValidationError):
        fio.geometry_from_dict({"variant": "helical", "n_views": 2, "n_detectors": 2})


def _cfg(tmp_path, **over):
    cfg = {"dims": [32, 32, 8],
           "geometry": {"variant": "parallel", "n_views": 12, "n_detectors": 48},
           "box": 9, "weights": "l1+ssim+tv", "optimizer": {"max_iters": 5},
           "init": {"mode": "fbp", "n_gaussians": 500, "seed": 0}}
    cfg.update(over)
    p = str(tmp_path / "run.json")
    json.dump(cfg, open(p, "w"))
    return p


def test_config_validation_exit_codes(tmp_path, capsys):
    out = str(tmp_path / "o")
    # missing sinogram path -> config error before any compute
    assert cli.main(["reconstruct", "--config", _cfg(tmp_path), "--out", out]) == 2
    assert cli.main(["reconstruct", "--config",
                     _cfg(tmp_path, paths={"sinogram": str(tmp_path / "nope.raw")}),
                     "--out", out]) == 2
    assert cli.main(["reconstruct", "--config", _cfg(tmp_path, weights="l2"), "--out", out]) == 2
    assert cli.main(["reconstruct", "--config", str(tmp_path / "missing.json"),
                     "--out", out]) == 2
    assert cli.main(["phantom", "--kind", "shepp-logan-3d", "--dims", "16", "16", "16",
                     "--out", out]) == 2          # dims >= 32 per axis
    st, geom, _ = cli.settings_from_config(cli.load_config(_cfg(tmp_path)))
    assert st.box.shape == (9, 9, 7) and st.max_iters == 5 and geom.n_views == 12


def test_phantom_command(tmp_path):
    p = str(tmp_path / "ph.raw")
    assert cli.main(["phantom", "--kind", "shepp-logan-3d", "--dims", "32", "32", "32",
                     "--out", p]) == 0
    assert fio.read_volume(p).zyx.tobytes() == phantom.shepp_logan_3d(32, 32, 32).zyx.tobytes()
    p2 = str(tmp_path / "ph2.raw")
    cli.main(["phantom", "--kind", "shepp-logan-3d", "--dims", "32", "32", "32", "--out", p2])
    assert open(p, "rb").read() == open(p2, "rb").read()          # deterministic


@pytest.mark.gpu
def test_metrics_command(tmp_path, capsys):
    p = str(tmp_path / "ph.raw")
    assert cli.main(["phantom", "--kind", "shepp-logan-3d", "--dims", "32", "32", "32",
                     "--out", p]) == 0
    capsys.readouterr()
    assert cli.main(["metrics", "--recon", p, "--truth", p]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["ssim_volume"] == pytest.approx(1.0) and rep["psnr_volume"] >= 200
    z = str(tmp_path / "z.raw")
    o = str(tmp_path / "o.raw")
    fio.write_volume(z, core.VolumeGrid.zeros((32, 32, 32)))
    fio.write_volume(o, core.VolumeGrid.from_zyx(np.full((32, 32, 32), 0.1, np.float32)))
    assert cli.main(["metrics", "--recon", o, "--truth", z, "--max", "1"]) == 0
    rep = json.loads(capsys.readouterr().out)
    assert rep["psnr_volume"] == pytest.approx(20.0, abs=1e-5)


@pytest.mark.gpu
def test_cli_project_reconstruct_pipeline(tmp_path, capsys):
    vol = str(tmp_path / "truth.raw")
    assert cli.main(["phantom", "--kind", "shepp-logan-3d", "--dims", "32", "32", "32",
                     "--out", vol]) == 0
    sino = str(tmp_path / "sino.raw")
    cfgp = _cfg(tmp_path, dims=[32, 32, 32])
    assert cli.main(["project", "--volume", vol, "--config", cfgp, "--out", sino]) == 0
    cfg = json.load(open(cfgp))
    cfg["paths"] = {"sinogram": sino, "truth": vol}
    json.dump(cfg, open(cfgp, "w"))
    out = str(tmp_path / "run")
    capsys.readouterr()
    assert cli.main(["reconstruct", "--config", cfgp, "--out", out]) == 0
    summary = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert summary["iterations"] == 5
    for f in ("volume.raw", "cloud.raw", "trace.csv"):
        assert os.path.exists(os.path.join(out, f))
    assert fio.read_cloud(os.path.join(out, "cloud.raw")).n == summary["n_gaussians"]
    fb = str(tmp_path / "fbp.raw")
    assert cli.main(["fbp", "--sinogram", sino, "--config", cfgp, "--out", fb]) == 0
    assert fio.read_volume(fb).dims == (32, 32, 32)
