"""Phase breakdown of optim.run_reconstruction at C2, as bench.py's e2e leg
calls it (GPU box helper; wrappers synchronise, so totals run slightly long).

    python tools/e2e_phases.py [--steps 50]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D, optim  # noqa: E402
from paper_2411_04844_b200.core import Sinogram  # noqa: E402

T = {}


def wrap(mod, name):
    fn = getattr(mod, name)

    def w(*a, **k):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = fn(*a, **k)
        torch.cuda.synchronize()
        T[name] = T.get(name, 0.0) + 1e3 * (time.perf_counter() - t0)
        return r
    setattr(mod, name, w)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=50)
    a = ap.parse_args()
    cfg = bench.CONFIGS["c2"]
    truth, geom, box, cloud = bench.make_problem(cfg)
    dev = torch.device("cuda", 0)
    w, h, c = cfg["dims"]
    op = D.projector_for(geom, w, h, 0.5, dev)
    meas = Sinogram.from_views(op.forward(D.zyx_to_yxz(truth.zyx, dev)).cpu().numpy())
    st = optim.ReconstructionSettings(dims=cfg["dims"], box=box, max_iters=a.steps,
                                      n_gaussians=cfg["n"], densify_interval=0)
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
        torch.cuda.synchronize()
        print(f"plain run {rep}: {1e3 * (time.perf_counter() - t0):.1f} ms")
    for name in ("cloud_to_params", "params_to_cloud", "to_pinned_host", "pinned_output",
                 "params_to_host", "cloud_from_host"):
        wrap(D, name)
    wrap(D.StagedHost, "__init__")
    wrap(optim, "_trainer_for")
    from paper_2411_04844_b200.trainer import Trainer
    wrap(D.StagedHost, "to")
    for name in ("initial_volume", "step", "trace_rows"):
        wrap(Trainer, name)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
    torch.cuda.synchronize()
    tot = 1e3 * (time.perf_counter() - t0)
    print(f"instrumented run: {tot:.1f} ms; " + ", ".join(f"{k} {v:.2f}" for k, v in T.items())
          + f"; not in a wrapper {tot - sum(T.values()):.2f}")


if __name__ == "__main__":
    main()
