"""Share of the TV epilogue in the C2 adjoint (GPU box helper): the training
step's adjoint (footprint-masked, TV fused) against the same call without TV,
CUDA-event medians of 20 launches each."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D, loss as L  # noqa: E402
from paper_2411_04844_b200.trainer import Trainer  # noqa: E402


def main():
    cfg = bench.CONFIGS["c2"]
    dev = torch.device("cuda", 0)
    truth, geom, box, cloud = bench.make_problem(cfg)
    w, h, c = cfg["dims"]
    op = D.operator_for(geom, w, h, c, 0.5, dev)
    meas = op.forward(D.zyx_to_yxz(np.ascontiguousarray(truth.zyx), dev))
    tr = Trainer(meas, geom, cfg["dims"], box, L.LossWeights(), D.cloud_to_params(cloud, dev),
                 max_iters=1000, trace_cap=64)
    tr.initial_volume()
    for _ in range(3):
        tr.iteration()
    torch.cuda.synchronize()
    lw = tr.weights
    dl = torch.empty_like(tr.dl)
    tv = torch.zeros_like(tr.tv_part)

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))
    with_tv = timed(lambda: tr.op.adjoint(tr.gpred, dl, vol=tr.vol, lambda_tv=lw.lambda3,
                                          tv_count=tr.tv_count, tv_partial=tv, halt=tr.halt,
                                          occ=tr.fvr))
    no_tv = timed(lambda: tr.op.adjoint(tr.gpred, dl, halt=tr.halt, occ=tr.fvr))
    dense = timed(lambda: tr.op.adjoint(tr.gpred, dl, halt=tr.halt))
    print(f"adjoint masked + TV {with_tv:.4f} ms, masked no TV {no_tv:.4f} ms, "
          f"dense no TV {dense:.4f} ms")


if __name__ == "__main__":
    main()
