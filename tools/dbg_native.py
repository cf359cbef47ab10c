import numpy as np, sys
sys.path.insert(0, "/root/repo")
from paper_2601_20782_b200 import rbm, F16, BF16, F32, RoundingMode
from paper_2601_20782_b200.precision import FORMATS
from oracle import model
g = np.load("tests/golden/forward.npz")
for ci in range(int(g["n_cases"])):
    p = rbm.RbmParameters(g[f"c{ci}_a"], g[f"c{ci}_b"], g[f"c{ci}_w"])
    bits = g[f"c{ci}_bits"]
    for fmt in ("f16", "bf16", "f32"):
        s = rbm.round_parameters(p, FORMATS[fmt])
        lp = rbm.log_prob_batch(p, bits, FORMATS[fmt], RoundingMode.NATIVE)
        want, tol = model.native_log_prob(s.a, s.b, s.w, bits, fmt)
        d = np.abs(lp - want)
        i = int(np.argmax(d - tol))
        print(ci, fmt, "max excess", (d - tol).max(), "row", i, lp[i], want[i], tol[i], "nbad", int((d > tol).sum()))
        if (d > tol).any():
            theta = bits[i].astype(float) @ s.w.T + s.b
            v = 1 + np.exp(-4*np.abs(theta.real)) + 2*np.exp(-2*np.abs(theta.real))*np.cos(2*theta.imag)
            print("   min v", v.min(), "theta at min", theta[np.argmin(v)])
