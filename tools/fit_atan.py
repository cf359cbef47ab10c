# Fits the atan polynomial used by atan2_fast in paper_2601_20782_b200/csrc/forward_tc.cu
# (degree 7 in s = a^2; prints the max f32-Horner error on [0,1] and the f32 coefficients).
import numpy as np
# fit atan(a)/a = p(s), s=a^2 on [0,1], degree D, weighted LS on Chebyshev nodes, then refine by IRLS toward minimax in absolute atan error
for D in (7,):
    n=4000
    s=(1-np.cos(np.pi*(np.arange(n)+0.5)/n))/2
    a=np.sqrt(s); f=np.where(a>0, np.arctan(a)/np.where(a>0,a,1),1.0)
    w=np.ones(n)
    for it in range(60):
        V=np.vander(s,D+1,increasing=True)*a[:,None]  # error in atan units
        c,*_=np.linalg.lstsq(V*w[:,None], (f*a)*w, rcond=None)
        e=np.abs(V@c-f*a); w*= (e/e.max()+1e-3)**0.3
    c32=c.astype(np.float32)
    # evaluate in f32 Horner
    x=np.linspace(0,1,2000001).astype(np.float32); s32=x*x
    p=np.float32(c32[-1])
    for k in range(D-1,-1,-1): p=(p*s32+c32[k]).astype(np.float32)
    r=(p*x).astype(np.float32)
    print(D, np.abs(r.astype(np.float64)-np.arctan(x.astype(np.float64))).max(), [float(v) for v in c32])
