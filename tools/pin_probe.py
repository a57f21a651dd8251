"""Host<->device copy paths for the e2e call: pinned staging + parallel host
copy (today) vs registering the caller's numpy buffer in place
(cudaHostRegister) and DMA-ing straight from / into it."""
import time
import numpy as np
import torch

cr = torch.cuda.cudart()


def t(fn, reps=3):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return min(ts)


for mb in (26, 64):
    n = mb * 262144
    a = np.random.rand(n).astype(np.float32)
    d = torch.empty(n, device="cuda")
    pin = torch.empty(n, pin_memory=True)

    def staged():
        np.copyto(pin.numpy(), a)
        d.copy_(pin, non_blocking=True)

    def reg():
        ptr = a.ctypes.data
        r = cr.cudaHostRegister(ptr, a.nbytes, 0)
        src = torch.from_numpy(a)
        d.copy_(src, non_blocking=True)
        torch.cuda.synchronize()
        cr.cudaHostUnregister(ptr)

    def reg_only():
        ptr = a.ctypes.data
        cr.cudaHostRegister(ptr, a.nbytes, 0)
        cr.cudaHostUnregister(ptr)

    def dma_pinned():
        d.copy_(pin, non_blocking=True)

    def pageable():
        d.copy_(torch.from_numpy(a))

    b = np.empty(n, np.float32)
    b.fill(0)

    def d2h_staged():
        pin.copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        np.copyto(b, pin.numpy())

    def d2h_reg():
        ptr = b.ctypes.data
        cr.cudaHostRegister(ptr, b.nbytes, 0)
        torch.from_numpy(b).copy_(d, non_blocking=True)
        torch.cuda.synchronize()
        cr.cudaHostUnregister(ptr)

    def d2h_pageable():
        torch.from_numpy(b).copy_(d)

    def h2d_pageable_chunks():
        k = 4
        step = (n + k - 1) // k
        for i in range(0, n, step):
            d[i:i + step].copy_(torch.from_numpy(a[i:i + step]), non_blocking=True)

    print(f"{mb} MB: pageable D2H {t(d2h_pageable):.2f} ms | pageable H2D 4 chunks "
          f"{t(h2d_pageable_chunks):.2f}", flush=True)
    print(f"{mb} MB: staged H2D {t(staged):.2f} ms | register+H2D+unregister {t(reg):.2f} | "
          f"register+unregister {t(reg_only):.2f} | pinned DMA {t(dma_pinned):.2f} | "
          f"pageable H2D {t(pageable):.2f} | staged D2H {t(d2h_staged):.2f} | "
          f"register D2H {t(d2h_reg):.2f}", flush=True)
