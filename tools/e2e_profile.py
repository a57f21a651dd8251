import os, sys, time
sys.path.insert(0, os.environ["GRAFT_REPO_ROOT"])
import numpy as np, torch
import bench
from paper_2411_04844_b200 import device as D, optim
from paper_2411_04844_b200.core import Sinogram
cfg = bench.CONFIGS["c2"]
truth, geom, box, cloud = bench.make_problem(cfg)
dev = torch.device("cuda", 0)
w, h, c = cfg["dims"]
op = D.projector_for(geom, w, h, 0.5, dev)
meas = Sinogram.from_views(op.forward(D.zyx_to_yxz(truth.zyx, dev)).cpu().numpy())
st = optim.ReconstructionSettings(dims=cfg["dims"], box=box, max_iters=int(os.environ.get("STEPS", "20")), densify_interval=0)
for _ in range(2): optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
import cProfile, pstats
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter(); optim.run_reconstruction(meas, geom, st, init_cloud=cloud); torch.cuda.synchronize()
print("total ms", 1e3*(time.perf_counter()-t0))
pr.disable(); pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
x = torch.empty((h, w, c), device=dev)
for name, fn in [("to_host", lambda: D.yxz_to_zyx(x)),
                 ("pageable", lambda: x.permute(2,0,1).contiguous().cpu().numpy()),
                 ]:
    fn(); torch.cuda.synchronize(); t0=time.perf_counter(); fn(); torch.cuda.synchronize(); print(name, 1e3*(time.perf_counter()-t0))
pin = torch.empty((c, h, w), pin_memory=True)
t0=time.perf_counter(); pin.copy_(x.permute(2,0,1).contiguous()); a = pin.numpy().copy(); print("cached pinned+copy", 1e3*(time.perf_counter()-t0))
t0=time.perf_counter(); pin.copy_(x.permute(2,0,1).contiguous()); print("cached pinned only", 1e3*(time.perf_counter()-t0))
t0=time.perf_counter(); a=np.empty((c,h,w),np.float32); torch.from_numpy(a).copy_(x.permute(2,0,1).contiguous()); print("into fresh pageable", 1e3*(time.perf_counter()-t0))
