"""Bins alone (footprints + sort + tile starts) for ncu launch lists.

    python tools/prof_bin.py --grid 256 --n 50000 [--reps 2]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2411_04844_b200 import core, device as D, optim  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--n", type=int, default=50_000)
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    dims = (a.grid,) * 3
    box = core.BoxConfig.for_dims(17, dims)
    cl = optim.init_cloud_random(dims, a.n, seed=0, box=box)
    dev = torch.device("cuda", 0)
    plan = D.FvrPlan(a.n, dims, box.half, 0, dev)
    params = D.cloud_to_params(cl, dev)
    for _ in range(a.reps):
        plan.bin(params)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
