"""Shared loader for tests/golden/densify.npz (the reference's own
densify_and_prune + OptimizerState.remap outputs, tests/golden/make_golden.py)."""
import os

import numpy as np

from paper_2411_04844_b200 import core, densify

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "densify.npz")


def cases():
    d = np.load(PATH)
    out = []
    for ci in range(int(d["d_ncases"])):
        g = {k[len(f"d{ci}_"):]: d[k] for k in d.files if k.startswith(f"d{ci}_")}
        n = g["mu"].shape[0]
        cloud = core.GaussianCloud(g["mu"], g["sigma"], g["intensity"])
        grads = core.ParamGradients(np.zeros((n, 3)), np.zeros(n), np.zeros(n), g["accum"],
                                    int(g["iters"]))
        prm = densify.DensifyParams(n_max=int(g["n_max"]), tau=float(g["tau"]),
                                    theta=float(g["theta"]), box_size=int(g["box"]),
                                    grad_prune_enabled=bool(g["grad_prune"]))
        out.append((ci, cloud, grads, prm, (int(g["seed"]), int(g["it"])), g))
    return out
