import os, sys
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import numpy as np, torch
import bench
from paper_2411_04844_b200 import device as D, loss as L
from paper_2411_04844_b200.trainer import Trainer
cfg = bench.CONFIGS["c2"]
truth, geom, box, cloud = bench.make_problem(cfg)
dev = torch.device("cuda", 0)
w, h, c = cfg["dims"]
op = D.operator_for(geom, w, h, c, 0.5, dev)
meas = op.forward(D.zyx_to_yxz(truth.zyx, dev))
tr = Trainer(meas, geom, cfg["dims"], box, L.LossWeights(), D.cloud_to_params(cloud, dev), max_iters=100, trace_cap=60)
tr.initial_volume()
for it in range(51):
    if it in (0, 50):
        pred = op.forward(tr.vol)
        for name, s in (("ref", meas), ("pred", pred), ("both", None)):
            if s is None:
                z = ((meas.abs().amax(0) == 0) & (pred.abs().amax(0) == 0))
            else:
                z = (s.abs().amax(0) == 0)        # (n_det, p): zero over all views
            zc = z.reshape(z.shape[0], -1, 32).all(-1)   # (n_det, p/32)
            n = zc.shape[0]
            # stats block: 7 output cols, 17 input cols starting at j0
            zs = zc.float().cpu().numpy()
            sk_s = np.mean([zs[j0:j0+17].min(0).mean() for j0 in range(0, n - 10, 7)])
            sk_g = np.mean([zs[max(s0-15,0):s0+12].min(0).mean() for s0 in range(0, n, 7)])
            print(it, name, "zero (d,z32) frac %.3f" % zs.mean(), "stats-block skip %.3f grad-block skip %.3f" % (sk_s, sk_g))
    tr.step()
