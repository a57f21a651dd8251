"""Eager C2 training iterations for profiling (ncu / compute-sanitizer).

    python tools/prof_step.py [--config c2] [--iters 3]

Sets up the bench workload (bench.make_problem) and runs a few eager
iterations (no CUDA graph) so every kernel launch is visible to ncu.
"""
import argparse
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
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--iters", type=int, default=3)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    truth, geom, box, cloud = bench.make_problem(cfg)
    dev = torch.device("cuda", 0)
    w, h, c = cfg["dims"]
    op = D.operator_for(geom, w, h, c, 0.5, dev)   # per-slice or cone
    meas = op.forward(D.zyx_to_yxz(np.ascontiguousarray(truth.zyx), dev))
    tr = Trainer(meas, geom, cfg["dims"], box, L.LossWeights(), D.cloud_to_params(cloud, dev),
                 max_iters=1000, trace_cap=a.iters + 1)
    tr.initial_volume()
    for _ in range(a.iters):
        tr.iteration()
    torch.cuda.synchronize()
    print("loss trace", tr.trace_rows()[:, 0], "nnz", getattr(op, "nnz", None))


if __name__ == "__main__":
    main()
