"""How much of the projector forward's gathered bytes are zero segments
(GPU box helper): at C2, the fraction of (entry, 128-slice chunk) gathers the
chunk-level skip keeps, and the fraction of their 16-slice segments that are
actually non-zero (what a per-segment skip would still read)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2411_04844_b200 import device as D, loss as L  # noqa: E402
from paper_2411_04844_b200.trainer import Trainer  # noqa: E402

cfg = bench.CONFIGS["c2"]
dev = torch.device("cuda", 0)
truth, geom, box, cloud = bench.make_problem(cfg)
w, h, c = cfg["dims"]
op = D.operator_for(geom, w, h, c, 0.5, dev)
meas = op.forward(D.zyx_to_yxz(np.ascontiguousarray(truth.zyx), dev))
tr = Trainer(meas, geom, cfg["dims"], box, L.LossWeights(), D.cloud_to_params(cloud, dev),
             max_iters=1000, trace_cap=64)
tr.initial_volume()
for _ in range(5):
    tr.iteration()
torch.cuda.synchronize()
words = tr.fvr.pixel_occupancy_words()[op.forward_entry_pixels().long()].cpu().numpy()
words = words.view(np.uint64)
ntz = c // 16
bits = ((words[:, None] >> np.arange(ntz, dtype=np.uint64)[None, :]) & np.uint64(1)).astype(bool)
chunks = bits.reshape(len(words), ntz // 8, 8)
kept = chunks.any(axis=2)
print("entries", len(words), "chunk gathers kept", kept.mean())
print("nonzero 16-slice segments among kept chunks", chunks[kept].mean())
print("overall nonzero segment fraction", bits.mean())
