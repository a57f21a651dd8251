"""The drop-in boundary: ``import splatct`` from ``pkg/src``
resolves to the B200 build, exposes the reference's public names and call
signatures (tests/golden/api_signatures.json, written by make_golden.py
--only api from the reference's own modules), and -- on the GPU -- replays
make_golden.py's reference call sequence through ``splatct.*`` against the
reference's outputs in kernels.npz.

Both run in a fresh interpreter whose only path entry for the package is
``pkg/src`` (reference: pkg/src/splatct/__init__.py:1-35).
"""
import json
import os
import subprocess
import sys

import pytest

from conftest import GOLDEN, ROOT

PKG_SRC = os.path.join(ROOT, "pkg", "src")


def _run(code, tmp_path):
    env = dict(os.environ)
    env["PYTHONPATH"] = PKG_SRC           # the repo root is NOT on the path
    r = subprocess.run([sys.executable, "-c", code], cwd=str(tmp_path), env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    return r.stdout


API_CHECK = r"""
import importlib, inspect, json, sys
import splatct
assert splatct.__file__.startswith(%(pkg)r), splatct.__file__
spec = json.load(open(%(spec)r))
missing = [n for n in spec["__all__"] if not hasattr(splatct, n)]
assert not missing, missing
for mod in ("core", "fvr", "projector", "loss", "optim", "densify", "metrics", "phantom"):
    m = importlib.import_module("splatct." + mod)
    assert m.__name__ == "paper_2411_04844_b200." + mod, m.__name__
    assert getattr(splatct, mod) is m
from splatct import fvr as f2
assert f2 is sys.modules["paper_2411_04844_b200.fvr"]
bad = []
for key, params in spec["signatures"].items():
    mod, qual = key.split(".", 1)
    obj = importlib.import_module("splatct." + mod)
    for part in qual.split("."):
        obj = getattr(obj, part)
    got = [[p.name, p.kind.name, p.default is not inspect.Parameter.empty]
           for p in inspect.signature(obj).parameters.values()]
    # the B200 build may append keyword arguments with defaults (cone fields)
    if got[:len(params)] != params or any(not d for _, _, d in got[len(params):]):
        bad.append((key, params, got))
assert not bad, bad
print("api ok", len(spec["signatures"]))
"""


def test_import_splatct_resolves_to_b200_build(tmp_path):
    out = _run(API_CHECK % {"pkg": PKG_SRC, "spec": os.path.join(GOLDEN, "api_signatures.json")},
               tmp_path)
    assert "api ok" in out


REPLAY = r"""
import numpy as np, warnings
import splatct
from splatct import core, fvr, projector, loss, optim
g = np.load(%(npz)r)
def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
cl = lambda p: core.GaussianCloud(g[p + "_mu"], g[p + "_sigma"], g[p + "_intensity"])
worst = {}
def note(k, v, tol):
    worst[k] = max(worst.get(k, 0.0), v)
    assert v < tol, (k, v)
with warnings.catch_warnings():
    warnings.simplefilter("ignore")
    for ci in range(int(g["fvr_ncases"])):
        dims = tuple(int(v) for v in g[f"fvr{ci}_dims"])
        box = core.BoxConfig(*(int(v) for v in g[f"fvr{ci}_box"]))
        vol = fvr.reconstruct(cl(f"fvr{ci}"), box, dims, deterministic=True)
        note("fvr.reconstruct", rel(vol.zyx, g[f"fvr{ci}_vol"]), 1e-5)
        gr = fvr.backward(cl(f"fvr{ci}"), box, dims, core.VolumeGrid.from_zyx(g[f"fvr{ci}_up"]))
        for k, ref in (("d_mu", "d_mu"), ("d_sigma", "d_sigma"),
                       ("d_intensity", "d_intensity"), ("accum_pos_grad_norm", "accum")):
            note("fvr.backward", rel(getattr(gr, k), g[f"fvr{ci}_{ref}"]), 1e-4)
for ci in range(int(g["proj_ncases"])):
    p = lambda k: g[f"proj{ci}_{k}"]
    ang = p("angles")
    if str(p("variant")) == "fan":
        geom = core.ScanGeometry("fan", len(ang), int(p("n_det")), float(p("spacing")), ang,
                                 float(p("rs")), float(p("rd")))
    else:
        geom = core.ScanGeometry("parallel", len(ang), int(p("n_det")), float(p("spacing")), ang)
    dims = tuple(int(v) for v in p("dims"))
    s = projector.forward_project(core.VolumeGrid.from_zyx(p("vol")), geom)
    note("projector.forward_project", rel(s.views, p("sino")), 1e-5)
    bp = projector.back_project(core.Sinogram.from_views(p("ys")), geom, dims, deterministic=True)
    note("projector.back_project", rel(bp.zyx, p("bp")), 1e-5)
for ci in range(int(g["loss_ncases"])):
    p = lambda k: g[f"loss{ci}_{k}"]
    v, gp, gv, parts = loss.total_loss_detailed(core.Sinogram.from_views(p("pred")),
                                                core.Sinogram.from_views(p("ref")),
                                                core.VolumeGrid.from_zyx(p("vol")),
                                                loss.LossWeights())
    note("loss.total_loss_detailed", abs(v - float(p("total"))), 1e-9)
    note("loss.grad_pred", rel(gp, p("grad_pred")), 1e-6)
    note("loss.grad_vol", rel(gv, p("grad_vol")), 1e-6)
c = core.GaussianCloud(g["adam_in_mu"], g["adam_in_sigma"], g["adam_in_intensity"])
gr = core.ParamGradients(g["adam_d_mu"], g["adam_d_sigma"], g["adam_d_intensity"],
                         np.zeros(len(g["adam_d_sigma"])), 1)
st = optim.OptimizerState(*(g[f"adam_in_{k}"] for k in ("m_mu", "v_mu", "m_sigma", "v_sigma",
                                                         "m_intensity", "v_intensity")),
                          int(g["adam_step"]), 3e-4, 3e-5, 100)
c2, s2 = optim.adam_step(c, gr, st, sigma_ceiling=51.0)
for k in ("mu", "sigma", "intensity"):
    note("optim.adam_step", rel(getattr(c2, k), g[f"adam_out_{k}"]), 1e-13)
import paper_2411_04844_b200._lib as L
assert L.load(build_if_missing=False) is not None
print("replay ok", worst)
"""


@pytest.mark.gpu
def test_reference_call_sequence_through_splatct(tmp_path):
    out = _run(REPLAY % {"npz": os.path.join(GOLDEN, "kernels.npz")}, tmp_path)
    assert "replay ok" in out
    print(out)
