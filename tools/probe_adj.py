"""Time the blocked adjoint at C2 with and without the fused TV epilogue."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D  # noqa: E402


def ms(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(True), torch.cuda.Event(True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


cfg = bench.CONFIGS["c2"]
truth, geom, box, cloud = bench.make_problem(cfg)
dev = torch.device("cuda", 0)
w, h, c = cfg["dims"]
op = D.projector_for(geom, w, h, 0.5, dev)
vol = D.zyx_to_yxz(truth.zyx, dev)
g = op.forward(vol)
out = torch.empty_like(vol)
part = torch.zeros(D.tv_partial_len(w, h, c), dtype=torch.float64, device=dev)
print("fwd", ms(lambda: op.forward(vol, g)))
print("adj no-tv", ms(lambda: op.adjoint(g, out)))
print("adj tv", ms(lambda: op.adjoint(g, out, vol=vol, lambda_tv=1.0, tv_count=float(w * h * c),
                                      tv_partial=part)))
print("fwd csr", ms(lambda: op.forward(vol, g, blocked=False)))
print("adj csr", ms(lambda: op.adjoint(g, out, blocked=False)))
