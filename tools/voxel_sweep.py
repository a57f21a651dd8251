"""Voxelize-only sweep (BASELINE.json configs[4]).

    python tools/voxel_sweep.py [--grids 128,256,512,1024] [--ns 10000,50000,400000,2000000]

For each (grid, N): init_cloud_random (sigma 1.5, box 17^3, unclipped), then
device times (CUDA events, median of 10 after 3 warm-ups) of
  bin   = footprints + radix sort + tile starts        (FvrPlan.bin)
  splat = the tile splat alone, on the binned cloud    (FvrPlan.forward)
  fwd   = bin + splat                                  (fvr.reconstruct)
  bwd   = the backward (gradients + norm accumulation; FvrPlan.backward,
          standard-normal upstream)
reported as voxel contributions/s and algorithmic HBM GB/s with their
fractions of the measured HBM peak and of the FP32 FMA peak (148 SMs x 128
lanes x sm clock).  Algorithmic bytes: splat 40 N + 4 W H C (params read,
volume written once); bwd 96 N + 4 min(C, W H C) -- the backward reads only
the upstream voxels inside footprints, each at most once, so a sparse cloud
in a large grid does not owe the whole upstream.  One JSON line per point.
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2411_04844_b200 import core, device as D, optim  # noqa: E402


def med_ms(fn, reps=10, warm=3):
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
    ap.add_argument("--grids", default="128,256,512,1024")
    ap.add_argument("--ns", default="10000,50000,400000,2000000")
    a = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else {"hbm_gbs": 6650.0,
                                                                           "sm_max_mhz": 1965.0}
    hbm = float(peaks["hbm_gbs"])
    fma = 148 * 128 * float(peaks.get("sm_max_mhz", 1965.0)) * 1e6
    dev = torch.device("cuda", 0)
    for g in (int(v) for v in a.grids.split(",")):
        dims = (g, g, g)
        box = core.BoxConfig.for_dims(17, dims)
        up = torch.randn((g, g, g), device=dev, generator=torch.Generator(device=dev).manual_seed(0))
        for n in (int(v) for v in a.ns.split(",")):
            cl = optim.init_cloud_random(dims, n, seed=0, box=box)
            params = D.cloud_to_params(cl, dev)
            plan = D.FvrPlan(n, dims, box.half, 0, dev)
            vol = plan.new_volume()
            grads = torch.empty((5, n), dtype=torch.float64, device=dev)
            accum = torch.zeros(n, dtype=torch.float64, device=dev)

            def fwd():
                plan.bin(params)
                plan.forward(params, vol)

            fwd()
            t_bin = med_ms(lambda: plan.bin(params))
            t_s = med_ms(lambda: plan.forward(params, vol))
            t_f = med_ms(fwd)
            t_b = med_ms(lambda: plan.backward(params, up, grads, accum))
            fl = np.floor(cl.mu)
            hv = np.array(box.half)
            span = np.minimum(fl + hv, g - 1) - np.maximum(fl - hv, 0) + 1
            contrib = int(np.prod(np.clip(span, 0, None), axis=1).sum())
            vb = 4.0 * g ** 3
            row = {"grid": g, "n": n, "contributions": contrib,
                   "bin_ms": round(t_bin, 4), "splat_ms": round(t_s, 4), "fwd_ms": round(t_f, 4),
                   "bwd_ms": round(t_b, 4),
                   "fwd_contrib_per_s": contrib / (t_f * 1e-3),
                   "splat_contrib_per_s": contrib / (t_s * 1e-3),
                   "bwd_contrib_per_s": contrib / (t_b * 1e-3),
                   "fwd_gbs": (40 * n + vb) / (t_f * 1e-3) / 1e9,
                   "splat_gbs": (40 * n + vb) / (t_s * 1e-3) / 1e9,
                   "bwd_gbs": (96 * n + 4.0 * min(contrib, g ** 3)) / (t_b * 1e-3) / 1e9}
            row["splat_hbm_frac"] = row["splat_gbs"] / hbm
            row["fwd_hbm_frac"] = row["fwd_gbs"] / hbm
            row["bwd_hbm_frac"] = row["bwd_gbs"] / hbm
            row["fwd_fma_frac"] = row["fwd_contrib_per_s"] / fma
            row["bwd_fma_frac"] = row["bwd_contrib_per_s"] / fma
            row["bound"] = "hbm" if contrib / (40 * n + vb) < fma / (hbm * 1e9) else "fp32"
            print(json.dumps(row), flush=True)
            del plan, vol, grads, accum, params
            torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
