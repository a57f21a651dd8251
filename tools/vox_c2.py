"""Voxelizer micro-benchmark on the headline cloud (bench.make_problem, C2 by
default): device medians of bin / forward / backward, plus a parity check of
each against the oracle at the same inputs.

    python tools/vox_c2.py [--config c2] [--reps 20] [--check]

Environment switches (SPLATCT_*) select kernel variants; each run prints one
JSON line so variants can be compared across invocations.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D  # noqa: E402


def med_ms(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(True), torch.cuda.Event(True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--check", action="store_true")
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    truth, geom, box, cloud = bench.make_problem(cfg)
    dev = torch.device("cuda", 0)
    dims = cfg["dims"]
    n = cloud.n
    params = D.cloud_to_params(cloud, dev)
    plan = D.FvrPlan(n, dims, box.half, 0, dev)
    vol = plan.new_volume()
    up = torch.randn(vol.shape, device=dev, generator=torch.Generator(device=dev).manual_seed(0))
    grads = torch.empty((5, n), dtype=torch.float64, device=dev)
    accum = torch.zeros(n, dtype=torch.float64, device=dev)
    plan.bin(params)
    t_bin = med_ms(lambda: plan.bin(params), a.reps)
    t_fwd = med_ms(lambda: plan.forward(params, vol, masks=True), a.reps)
    t_bwd = med_ms(lambda: plan.backward(params, up, grads, accum), a.reps)
    out = {"config": a.config, "n": n, "bin_ms": round(t_bin, 4), "fwd_ms": round(t_fwd, 4),
           "bwd_ms": round(t_bwd, 4),
           "env": {k: v for k, v in os.environ.items() if k.startswith("SPLATCT_")}}
    if a.check:
        from oracle import oracle as O
        rel = lambda x, y: float(np.linalg.norm(x - y) / np.linalg.norm(y))
        plan.forward(params, vol, masks=True)
        ovol = O.splat_fwd(cloud.mu, cloud.sigma, cloud.intensity, box.shape, dims)
        out["fwd_rel_l2"] = rel(D.yxz_to_zyx(vol).astype(np.float64), ovol)
        accum.zero_()
        plan.backward(params, up, grads, accum)
        upz = D.yxz_to_zyx(up)
        dm, ds, di, acc, _ = O.splat_bwd(cloud.mu, cloud.sigma, cloud.intensity, box.shape, dims,
                                         upz)
        g = grads.cpu().numpy()
        out["bwd_rel_l2"] = max(rel(g[0:3].T, dm), rel(g[3], ds), rel(g[4], di))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
