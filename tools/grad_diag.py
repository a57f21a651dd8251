"""First-iteration gradient of the device step vs the oracle on the reference's
C2 pin problem (256^3 Shepp-Logan, fan 50x512, reference FBP-init cloud),
with the measured sinogram from the oracle or from the device projector;
per-term breakdown (L1 only, SSIM only, TV only)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2411_04844_b200 import core, device as D, loss, phantom, projector
from paper_2411_04844_b200.trainer import Trainer

g = np.load("tests/golden/c2pins.npz")
dims = (256, 256, 256)
truth = phantom.shepp_logan_3d(*dims)
og = O.Geometry.fan(50, 512, 1.6, 512.0, 512.0)
geom = core.ScanGeometry.fan(50, 512, 1.6, 512.0, 512.0)
box = core.BoxConfig.for_dims(17, dims)
mu, sg, it = g["c2p50_init_mu"], g["c2p50_init_sigma"], g["c2p50_init_intensity"]
meas_o = O.project_forward(truth.zyx, og)
meas_d = projector.forward_project(truth, geom).views
print("meas rel", np.linalg.norm(meas_d - meas_o) / np.linalg.norm(meas_o), flush=True)
dev = torch.device("cuda", 0)
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
v = O.splat_fwd(mu, sg, it, box.shape, dims)
pred = O.project_forward(v, og)
for lam in ((0.6, 0.2, 1.0), (1.0, 0.0, 0.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0)):
    _, gp, gv, _ = O.total_loss_detailed(pred, meas_o, v, lam)
    dl = (O.project_adjoint(gp.astype(np.float32), og, dims).astype(np.float64) + gv)
    dm, ds, di, _, _ = O.splat_bwd(mu, sg, it, box.shape, dims, dl.astype(np.float32))
    for name, meas in (("oracle meas", meas_o), ("device meas", meas_d)):
        tr = Trainer(torch.from_numpy(np.ascontiguousarray(meas)).to(dev), geom, dims, box,
                     loss.LossWeights(*lam), D.cloud_to_params(core.GaussianCloud(mu, sg, it), dev),
                     max_iters=4, trace_cap=2)
        tr.initial_volume()
        tr.iteration()
        torch.cuda.synchronize()
        gd = tr.grads.cpu().numpy()
        print(lam, name, "d_mu", rel(gd[0:3].T, dm), "d_sigma", rel(gd[3], ds), "d_I", rel(gd[4], di), flush=True)
