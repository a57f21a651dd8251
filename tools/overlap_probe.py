"""Do the step's stages overlap when run on two streams?  (C2, GPU box helper.)

Times, with CUDA events around a fork/join, pairs of independent stage
launches run back to back on one stream and concurrently on two streams:
  proj_forward || loss      (loss on a second prediction buffer)
  loss || proj_adjoint_tv   (adjoint of a second gradient buffer)
  proj_forward || proj_adjoint_tv
A concurrent time well under the sequential sum says a z-chunk software
pipeline of project -> loss -> adjoint would pay.

    python tools/overlap_probe.py
"""
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
    pred2, gpred2 = tr.pred.clone(), tr.gpred.clone()
    dl2 = torch.empty_like(tr.dl)
    tv2 = torch.zeros_like(tr.tv_part)
    sums2 = torch.zeros_like(tr.sums)
    loss2 = D.LossPlan(tr.m, tr.n, tr.pred.shape[2], dev)
    loss2.prepare(tr.meas)

    def proj():
        tr.op.forward(tr.vol, tr.pred, tr.halt, occ=tr.fvr)

    def lossf():
        loss2.fused(pred2, tr.meas, tr.lmax, lw.lambda1, lw.lambda2, tr.l1_count,
                    float(c), tr.gpred, sums2, tr.halt)

    def adj():
        tr.op.adjoint(gpred2, dl2, vol=tr.vol, lambda_tv=lw.lambda3, tv_count=tr.tv_count,
                      tv_partial=tv2, halt=tr.halt, occ=tr.fvr)

    s0 = torch.cuda.current_stream()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s0)
            fn()
            b.record(s0)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.median(ts))

    def conc(f, g):
        def run():
            s1.wait_stream(s0)
            s2.wait_stream(s0)
            with torch.cuda.stream(s1):
                f()
            with torch.cuda.stream(s2):
                g()
            s0.wait_stream(s1)
            s0.wait_stream(s2)
        return run

    single = {"proj": timed(proj), "loss": timed(lossf), "adj": timed(adj)}
    print("single", {k: round(v, 4) for k, v in single.items()})
    for a, b in (("proj", "loss"), ("loss", "adj"), ("proj", "adj")):
        fa, fb = {"proj": proj, "loss": lossf, "adj": adj}[a], {"proj": proj, "loss": lossf,
                                                                  "adj": adj}[b]
        seq = timed(lambda: (fa(), fb()))
        par = timed(conc(fa, fb))
        print(f"{a}+{b}: sequential {seq:.4f} ms, two streams {par:.4f} ms "
              f"(saving {100 * (1 - par / seq):.0f} %)")


if __name__ == "__main__":
    main()
