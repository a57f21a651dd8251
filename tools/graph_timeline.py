"""Kernel timeline of graph-replayed C2 iterations (torch.profiler / CUPTI):
per kernel start offset, duration and the idle gap before it, so launch
gaps between the step's kernels are visible (GPU box helper).

    python tools/graph_timeline.py
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
    tr.capture()
    for _ in range(5):
        tr.step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(3):
            tr.step()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    ev.sort(key=lambda e: e.time_range.start)
    t0 = ev[0].time_range.start
    prev_end = t0
    gaps = 0.0
    for e in ev:
        s, d = e.time_range.start, e.time_range.elapsed_us()
        gap = s - prev_end
        gaps += max(gap, 0)
        print(f"{s - t0:9.1f} us  dur {d:7.1f}  gap {gap:6.1f}  {e.name[:60]}")
        prev_end = max(prev_end, s + d)
    span = prev_end - t0
    print(f"span {span:.1f} us for 3 iterations, idle {gaps:.1f} us ({100 * gaps / span:.1f} %)")


if __name__ == "__main__":
    main()
