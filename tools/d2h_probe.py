"""D2H bandwidth of the 64 MB output volume: one copy vs chunks on 1 / 2 / 4
streams into page-locked memory (GPU box helper)."""
import time

import torch

n = 64 << 18   # 64 MB of f32
d = torch.rand(n, device="cuda")
h = torch.empty(n, pin_memory=True)
streams = [torch.cuda.Stream() for _ in range(4)]


def run(k, ns):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    step = n // k
    main = torch.cuda.current_stream()
    for i in range(k):
        s = streams[i % ns] if ns > 1 else main
        s.wait_stream(main)
        with torch.cuda.stream(s):
            h[i * step:(i + 1) * step].copy_(d[i * step:(i + 1) * step], non_blocking=True)
    for s in streams[:ns]:
        main.wait_stream(s)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for k, ns in ((1, 1), (2, 2), (4, 4), (8, 2), (8, 4), (16, 4)):
    ts = sorted(run(k, ns) for _ in range(7))
    print(f"{k} chunks on {ns} streams: {1e3 * ts[3]:.3f} ms, {n * 4 / ts[3] / 1e9:.1f} GB/s")
