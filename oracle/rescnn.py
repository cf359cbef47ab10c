"""numpy f64 restatement of the ResCNN neural quantum state — test infrastructure only.

The reference package has no convolutional ansatz; the model is specified by
the paper only (used at PAPER.md:301 for
configs[3]).  Parity for it is therefore UNPINNED by reference code: this
restatement is the spec the device kernels are checked against, plus exact
H psi on enumerable lattices.

    s = 1 - 2 x                                  (spins, one input channel)
    h0 = Conv(s)                                 (embedding, F filters)
    h_{l+1} = h_l + Conv(GELU(Conv(GELU(LN(h_l)))))   l = 0 .. n_res - 1
    log psi(x) = sum_{sites, channels} LN(h_{n_res})

Convolutions are K x K (K = 3), periodic, with bias; LN normalises the F
channels of each site (eps 1e-6) with a learned gain and shift; GELU is the
tanh form.  log psi is real (log p = 2 log psi).
"""
from __future__ import annotations

import numpy as np

LN_EPS = 1e-6


def param_shapes(filters: int, n_res: int, kernel: int = 3):
    """(name, shape) in the flattened parameter order."""
    F, T = filters, kernel * kernel
    out = [("w0", (F, 1, T)), ("b0", (F,))]
    for i in range(n_res):
        out += [(f"g{i}", (F,)), (f"be{i}", (F,)), (f"w{i}a", (F, F, T)), (f"b{i}a", (F,)),
                (f"w{i}b", (F, F, T)), (f"b{i}b", (F,))]
    out += [("gf", (F,)), ("bef", (F,))]
    return out


def unflatten(theta, filters, n_res, kernel=3):
    out, k = {}, 0
    for name, shape in param_shapes(filters, n_res, kernel):
        size = int(np.prod(shape))
        out[name] = np.asarray(theta[k:k + size], dtype=np.float64).reshape(shape)
        k += size
    return out


def _conv(h, w, b, L, kernel):
    """h [B, L*L, Cin], w [Cout, Cin, K*K] -> [B, L*L, Cout] (periodic)."""
    B = h.shape[0]
    hh = h.reshape(B, L, L, -1)
    out = np.zeros((B, L, L, w.shape[0]))
    r = kernel // 2
    for dy in range(-r, r + 1):
        for dx in range(-r, r + 1):
            tap = (dy + r) * kernel + (dx + r)
            shifted = np.roll(hh, shift=(-dy, -dx), axis=(1, 2))  # shifted[y, x] = hh[y + dy, x + dx]
            out += shifted @ w[:, :, tap].T
    return (out + b).reshape(B, L * L, -1)


def _ln(h, g, be):
    mu = h.mean(axis=-1, keepdims=True)
    var = ((h - mu) ** 2).mean(axis=-1, keepdims=True)
    return g * (h - mu) / np.sqrt(var + LN_EPS) + be


def gelu(z):
    return 0.5 * z * (1.0 + np.tanh(np.sqrt(2.0 / np.pi) * (z + 0.044715 * z ** 3)))


def log_psi(theta, bits, L, filters, n_res, kernel=3):
    """log psi for a (B, L*L) 0/1 matrix (row-major sites)."""
    p = unflatten(theta, filters, n_res, kernel)
    s = (1.0 - 2.0 * np.asarray(bits, dtype=np.float64))[:, :, None]
    h = _conv(s, p["w0"], p["b0"], L, kernel)
    for i in range(n_res):
        u = gelu(_ln(h, p[f"g{i}"], p[f"be{i}"]))
        v = gelu(_conv(u, p[f"w{i}a"], p[f"b{i}a"], L, kernel))
        h = h + _conv(v, p[f"w{i}b"], p[f"b{i}b"], L, kernel)
    return _ln(h, p["gf"], p["bef"]).sum(axis=(1, 2))
