"""Cone-beam projector pair at the C2-cone size, for ncu.

    python tools/prof_cone.py [--reps 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    cfg = bench.CONFIGS["c2cone"]
    truth, geom, box, cloud = bench.make_problem(cfg)
    dev = torch.device("cuda", 0)
    w, h, c = cfg["dims"]
    op = D.ConeOperator(geom, w, h, c, 0.5, dev)
    vol = D.zyx_to_yxz(np.ascontiguousarray(truth.zyx), dev)
    out = torch.empty((h, w, c), dtype=torch.float32, device=dev)
    for _ in range(a.reps):
        p = op.forward(vol)
        op.adjoint(p, out, c_local=c)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    p = op.forward(vol)
    ev[1].record()
    op.adjoint(p, out, c_local=c)
    ev[2].record()
    torch.cuda.synchronize()
    print("samples", op.n_samples, "entries", op.n_entries, "fwd ms", ev[0].elapsed_time(ev[1]),
          "adj ms", ev[1].elapsed_time(ev[2]))


if __name__ == "__main__":
    main()
