"""TV sign-subgradient sensitivity on the reference's C2 pin problem (CPU,
oracle): perturb the oracle's own splatted volume by 2e-7 relative noise and
report how far the TV part of the parameter gradients moves (DESIGN.md
section 2, "Sign-subgradient sensitivity").

    python tools/tv_sensitivity.py
"""
import numpy as np, sys
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from oracle import oracle as O
g=np.load(__import__('os').path.join(sys.path[0], 'tests', 'golden', 'c2pins.npz'))
dims=(256,256,256)
mu,sg,it=g['c2p50_init_mu'],g['c2p50_init_sigma'],g['c2p50_init_intensity']
v=O.splat_fwd(mu,sg,it,(17,17,17),dims)
rng=np.random.default_rng(0)
vp=(v.astype(np.float64)*(1+2e-7*rng.standard_normal(v.shape))).astype(np.float32)
print('vol rel', np.linalg.norm(vp-v)/np.linalg.norm(v))
res=[]
for vol in (v, vp):
    tv, gv = O.tv_loss(vol)
    dm,ds,di,_,_=O.splat_bwd(mu,sg,it,(17,17,17),dims,gv.astype(np.float32))
    res.append((dm,ds,di))
rel=lambda a,b: np.linalg.norm(a-b)/np.linalg.norm(b)
print('TV-only gradient change from a 2e-7 volume perturbation: d_mu', rel(res[1][0],res[0][0]), 'd_sigma', rel(res[1][1],res[0][1]), 'd_I', rel(res[1][2],res[0][2]))
tv, gv = O.tv_loss(v); tvp, gvp = O.tv_loss(vp)
print('tv grad entries changed', int((gv!=gvp).sum()), 'of', gv.size)
