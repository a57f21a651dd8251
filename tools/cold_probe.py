"""Cold run_reconstruction calls at C2 (after optim.clear_caches()): wall time
of three cold calls and of the operator build alone (GPU box helper).

    python tools/cold_probe.py
"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D, optim  # noqa: E402
from paper_2411_04844_b200.core import Sinogram  # noqa: E402


def main():
    cfg = bench.CONFIGS["c2"]
    truth, geom, box, cloud = bench.make_problem(cfg)
    dev = torch.device("cuda", 0)
    w, h, c = cfg["dims"]
    op = D.projector_for(geom, w, h, 0.5, dev)
    meas = Sinogram.from_views(op.forward(D.zyx_to_yxz(truth.zyx, dev)).cpu().numpy())
    st = optim.ReconstructionSettings(dims=cfg["dims"], box=box, max_iters=20, densify_interval=0)
    optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
    for k in range(3):
        optim.clear_caches()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
        torch.cuda.synchronize()
        print(f"cold call {k}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    optim.clear_caches()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    D.projector_for(geom, w, h, 0.5, dev)
    torch.cuda.synchronize()
    print(f"operator build: {1e3 * (time.perf_counter() - t0):.1f} ms")
    # phase split of one cold call (each wrapper synchronises)
    from paper_2411_04844_b200.trainer import Trainer
    T = {}

    def wrap(obj, name):
        fn = getattr(obj, name)

        def w_(*a, **k):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            r = fn(*a, **k)
            torch.cuda.synchronize()
            T[name] = T.get(name, 0.0) + 1e3 * (time.perf_counter() - t1)
            return r
        setattr(obj, name, w_)
    wrap(D, "operator_for")
    wrap(Trainer, "__init__")
    wrap(Trainer, "capture")
    wrap(Trainer, "initial_volume")
    wrap(Trainer, "step")
    optim.clear_caches()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
    torch.cuda.synchronize()
    print(f"cold call {1e3 * (time.perf_counter() - t0):.1f} ms: " +
          ", ".join(f"{k} {v:.2f}" for k, v in T.items()))


if __name__ == "__main__":
    main()
