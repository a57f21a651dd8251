"""Quick device timing probe for individual stages (GPU box helper)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D, loss as L, optim  # noqa: E402
from paper_2411_04844_b200.core import Sinogram  # noqa: E402


def timeit(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    truth, geom, box, cloud = bench.make_problem(cfg)
    dev = torch.device("cuda", 0)
    w, h, c = cfg["dims"]
    t0 = time.perf_counter()
    op = D.ProjectorOperator(geom, w, h, 0.5, dev)
    torch.cuda.synchronize()
    print(f"operator build {time.perf_counter() - t0:.3f} s; nnz {op.nnz} fwd-blocks {op.fb[3]} "
          f"adj-blocks {op.ab[3]}")
    vol = D.zyx_to_yxz(truth.zyx, dev)
    sino = op.forward(vol)
    print("fwd blocked ms", timeit(lambda: op.forward(vol, sino, blocked=True)))
    print("fwd csr ms", timeit(lambda: op.forward(vol, sino, blocked=False)))
    out = torch.empty_like(vol)
    part = torch.empty(w * h, dtype=torch.float64, device=dev)
    for bl in (True, False):
        print("adj+tv blocked" if bl else "adj+tv csr", "ms",
              timeit(lambda: op.adjoint(sino, out, vol=vol, lambda_tv=1.0, tv_count=float(vol.numel()),
                                        tv_partial=part, blocked=bl)))
        print("adj plain blocked" if bl else "adj plain csr", "ms",
              timeit(lambda: op.adjoint(sino, out, blocked=bl)))
    meas = Sinogram.from_views(sino.cpu().numpy())
    st = optim.ReconstructionSettings(dims=cfg["dims"], box=box, max_iters=30, densify_interval=0)
    for k in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
        torch.cuda.synchronize()
        print(f"run_reconstruction 30 iters: {time.perf_counter() - t0:.3f} s")


if __name__ == "__main__":
    main()
