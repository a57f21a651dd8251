"""Cost of densification events in run_reconstruction at C2 (GPU box helper)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D, optim  # noqa: E402
from paper_2411_04844_b200.core import Sinogram  # noqa: E402

cfg = bench.CONFIGS["c2"]
truth, geom, box, cloud = bench.make_problem(cfg)
dev = torch.device("cuda", 0)
w, h, c = cfg["dims"]
op = D.projector_for(geom, w, h, 0.5, dev)
meas = Sinogram.from_views(op.forward(D.zyx_to_yxz(truth.zyx, dev)).cpu().numpy())
for interval in (0, 100):
    st = optim.ReconstructionSettings(dims=cfg["dims"], box=box, max_iters=300,
                                      n_gaussians=cfg["n"], densify_interval=interval)
    optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    vol, cl, tr = optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    ev = [(r.iteration, r.clones, r.splits, r.prunes, r.n_gaussians) for r in tr if r.clones or r.splits or r.prunes]
    print(f"interval {interval}: {dt*1e3:.1f} ms for 300 its ({300/dt:.1f} it/s), final N {cl.n}, events {ev}")
