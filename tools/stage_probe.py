"""Where the measured sinogram's staging time goes inside run_reconstruction
(GPU box helper): join wait vs upload, per warm call (PREALLOC=1: upload into
a preallocated device buffer).  Finding: the 26 MB pinned -> device copy runs
at ~18 GB/s right after the host threads wrote the pinned pages, against
~45 GB/s for pages not written recently (tools/pin_probe.py)."""
import os
import sys
import time

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D, optim  # noqa: E402
from paper_2411_04844_b200.core import Sinogram  # noqa: E402

orig_init, orig_to = D.StagedHost.__init__, D.StagedHost.to
log = []


def init(self, views, device):
    self._t0 = time.perf_counter()
    orig_init(self, views, device)


def to(self, device):
    t1 = time.perf_counter()
    self._th.join()
    t2 = time.perf_counter()
    if os.environ.get("PREALLOC"):
        global _buf
        if "_buf" not in globals():
            _buf = torch.empty(self.a.shape, dtype=torch.float32, device=device)
        out = _buf.copy_(self.st.view(self.a.shape), non_blocking=True)
    else:
        out = orig_to(self, device)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    log.append((1e3 * (t1 - self._t0), 1e3 * (t2 - t1), 1e3 * (t3 - t2)))
    return out


D.StagedHost.__init__, D.StagedHost.to = init, to
cfg = bench.CONFIGS["c2"]
truth, geom, box, cloud = bench.make_problem(cfg)
dev = torch.device("cuda", 0)
w, h, c = cfg["dims"]
op = D.projector_for(geom, w, h, 0.5, dev)
meas = Sinogram.from_views(op.forward(D.zyx_to_yxz(truth.zyx, dev)).cpu().numpy())
st = optim.ReconstructionSettings(dims=cfg["dims"], box=box, max_iters=20, densify_interval=0)
for _ in range(5):
    optim.run_reconstruction(meas, geom, st, init_cloud=cloud)
for a, b, u in log:
    print(f"before join {a:.2f} ms, join wait {b:.2f} ms, upload {u:.2f} ms")
print("views flags", meas.views.flags["C_CONTIGUOUS"], meas.views.dtype, meas.views.shape)
