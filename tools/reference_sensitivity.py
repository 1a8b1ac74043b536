"""Sensitivity of the REFERENCE algorithm (oracle port, bitwise equal to the reference at cfg2)
to ulp-level perturbations: mode noise = 1e-16 relative noise on f(0); mode inv = the Poisson
solve by the explicit inverse (this build's method) instead of LU.  Compares with
tests/golden/coeffs_cfg2.npz after 1, 5, 50 steps (build container only; ~10 min).
"""
import sys, json, numpy as np
sys.path.insert(0,'/root/repo')
from oracle import sldg_oracle as so
mode=sys.argv[1]
g=np.load('/root/repo/tests/golden/coeffs_cfg2.npz')
sim=so.Sim(dim=3,n_base=32,levels=0,degree=2,n_x=64,workers=4)
if mode=='noise':
    rng=np.random.default_rng(1)
    sim.f *= 1.0 + 1e-16*rng.standard_normal(sim.f.shape)
elif mode=='inv':
    P=sim.poisson
    G=np.linalg.inv(P.aug)[:P.nn,:P.nn]
    P.solve=lambda r: G @ P.rhs(r)
for n in range(1,51):
    sim.step()
    if n in (1,5,50):
        f=sim.f.ravel()[g['sample_idx']]; ref=g[f's{n}_val']; fmax=float(g[f's{n}_fmax'])
        err=np.abs(f-ref); out={'mode':mode,'step':n,'normwise':err.max()/fmax}
        for thr in (1e-3,1e-2,1e-1):
            big=np.abs(ref)>=thr*fmax; out[f'rel@{thr:g}']=float((err[big]/np.abs(ref[big])).max())
        print(json.dumps(out),flush=True)
