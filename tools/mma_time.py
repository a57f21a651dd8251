import torch, numpy as np, sys
sys.path.insert(0,'.')
from paper_2411_04844_b200 import device as D
dev = D.require_cuda()
for two in (False, True):
    for nm in (2, 64, 512, 4096):
        a = torch.zeros((128, 8), device=dev); a[0,0] = 1000.0 if two else 0.0
        b = torch.zeros((16, 8), device=dev); d = torch.zeros((128, 16), device=dev)
        D.call("splatct_tc_selftest", D.ptr(a), D.ptr(b), D.ptr(d), nm, D.stream_handle())
        torch.cuda.synchronize()
        print("two" if two else "one", nm, "cycles", d[0,0].item(), "per mma", d[0,0].item()/nm)
