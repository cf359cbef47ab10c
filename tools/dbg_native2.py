import numpy as np, sys
sys.path.insert(0, "/root/repo")
from paper_2601_20782_b200 import rbm, F16, RoundingMode
from paper_2601_20782_b200.precision import FORMATS
from oracle import model
g = np.load("tests/golden/forward.npz")
ci = 0
p = rbm.RbmParameters(g[f"c{ci}_a"], g[f"c{ci}_b"], g[f"c{ci}_w"])
bits = g[f"c{ci}_bits"][:8]
s = rbm.round_parameters(p, F16)
ev = rbm.log_prob_evaluator(p, F16, RoundingMode.NATIVE)
print(ev.snapshot.label, rbm.plan_exact(s))
lp = ev(bits)
want, tol = model.native_log_prob(s.a, s.b, s.w, bits, "f16")
theta = bits.astype(float) @ s.w.T + s.b
lc = model.re_logcosh(theta.real, theta.imag)
vis = bits.astype(float) @ s.a.real
for r in range(8):
    print(r, "diff/2", (lp[r]-want[r])/2, "vis", vis[r], "lc", np.round(lc[r], 4), "bits", bits[r])
