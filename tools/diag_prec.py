import numpy as np
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
from spectra import full_from_half, half_spectrum
import torch
from oracle import dbfft_oracle as O
from synth import microstructure as ms
from paper_1905_12725_b200 import dbfft as dbf
n=(32,128,256)
u = ms.SplitMix64(21).uniform(n[0]*n[1]*n[2]).reshape(n[2],n[1],n[0]); ph=(u<0.3).astype(np.uint16)
ISO2 = [dict(kind="iso", E=1.0, nu=0.3), dict(kind="iso", E=10.0, nu=0.25)]
r=ms.random_field((3,n[2],n[1],n[0]),22)
C=O.stiffness_field(ph, ISO2)
zref=O.precondition(O.fft(r), C.mean(axis=(-3,-2,-1)), O.frequency_grid(n))
for P in (1,2):
    kw=dict(world=P, loopback=True) if P>1 else {}
    ctx=dbf.DBFFT(n, kinematics="small", **kw); ctx.set_phases(ph, ISO2)
    z=full_from_half(ctx.precond(torch.from_numpy(half_spectrum(r)).cuda()).cpu().numpy(), n[0])
    d=np.abs(z-zref).sum(axis=0); 
    print(P, 'rel', np.linalg.norm(z-zref)/np.linalg.norm(zref), 'max abs', d.max(), 'at', np.unravel_index(d.argmax(), d.shape), 'ref there', np.abs(zref).sum(axis=0)[np.unravel_index(d.argmax(), d.shape)])
    # relative error per point
    rr=d/np.maximum(np.abs(zref).sum(axis=0),1e-300)
    print('   max pointwise rel', rr.max(), np.unravel_index(rr.argmax(), rr.shape))
