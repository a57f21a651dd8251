"""Break down optim.run_reconstruction's fixed overhead at C2 (GPU box helper)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D, optim  # noqa: E402
from paper_2411_04844_b200.core import Sinogram  # noqa: E402
from paper_2411_04844_b200.loss import LossWeights  # noqa: E402
from paper_2411_04844_b200.trainer import Trainer  # noqa: E402


def t():
    torch.cuda.synchronize()
    return time.perf_counter()


def main():
    cfg = bench.CONFIGS["c2"]
    truth, geom, box, cloud = bench.make_problem(cfg)
    dev = torch.device("cuda", 0)
    w, h, c = cfg["dims"]
    op = D.projector_for(geom, w, h, 0.5, dev)
    meas_dev = op.forward(D.zyx_to_yxz(truth.zyx, dev))
    meas = Sinogram.from_views(meas_dev.cpu().numpy())
    st = optim.ReconstructionSettings(dims=cfg["dims"], box=box, max_iters=30, densify_interval=0)
    for rep in range(3):
        t0 = t()
        m_dev = D.sino_to_device(meas.views, dev)
        t1 = t()
        params = D.cloud_to_params(cloud, dev)
        st0 = optim.OptimizerState.fresh(cloud.n)
        m1, m2 = st0.moments_to_device(dev)
        t2 = t()
        tr = Trainer(m_dev, geom, cfg["dims"], box, LossWeights(), params, m1=m1, m2=m2,
                     max_iters=30, trace_cap=30)
        t3 = t()
        tr.initial_volume()
        t4 = t()
        tr.capture()
        t5 = t()
        for _ in range(29):
            tr.step()
        t6 = t()
        rows = tr.trace.cpu().numpy()
        vol = D.yxz_to_zyx(tr.vol)
        cl = D.params_to_cloud(tr.params)
        t7 = t()
        print(f"rep {rep}: h2d {1e3*(t1-t0):.1f} ms, params {1e3*(t2-t1):.1f}, trainer {1e3*(t3-t2):.1f}, "
              f"init-vol {1e3*(t4-t3):.1f}, capture(+1 iter) {1e3*(t5-t4):.1f}, 29 iters {1e3*(t6-t5):.1f}, "
              f"d2h {1e3*(t7-t6):.1f}, total {1e3*(t7-t0):.1f}")
        t0 = t()
        optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
        print(f"      run_reconstruction total {1e3*(t()-t0):.1f} ms")


if __name__ == "__main__":
    main()
