"""numpy models of the device arithmetic — test infrastructure only.

native_log_prob: the NATIVE-mode log p the fused sweep computes:
theta = b + W x exact (float64 sums of fmt-grid values are exact here), rounded
once to the format (via f32, double rounding is innocuous for p <= 24), each
unit's Re log cosh evaluated accurately and rounded to the format, summed in
f32, plus the exactly accumulated visible term rounded to f32, doubled.  The
device evaluates log cosh with MUFU approximations (|err| ~ 2e-7) and sums in a
lane-dependent order, so device == model within a per-row tolerance returned
alongside (one format ulp per unit plus 1e-6 per unit).
"""
from __future__ import annotations

import numpy as np

_ROUND = {
    "f16": lambda v: v.astype(np.float32).astype(np.float16).astype(np.float64),
    "f32": lambda v: v.astype(np.float32).astype(np.float64),
}


def _round(v, fmt):
    if fmt == "bf16":
        f = np.asarray(v, dtype=np.float32)
        u = f.view(np.uint32).astype(np.uint64)
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
        return u.astype(np.uint32).view(np.float32).astype(np.float64)
    return _ROUND[fmt](np.asarray(v, dtype=np.float64))


def re_logcosh(x, y):
    """Re log cosh(x + iy), accurate f64 (same closed form as ref rbm.py:130-140)."""
    u = np.abs(x)
    t = np.exp(-2.0 * u)
    return u - np.log(2.0) + 0.5 * np.log1p(t * t + 2.0 * t * np.cos(2.0 * y))


def native_log_prob(a, b, w, bits, fmt):
    """(lp_model, tol) for rows of `bits`; a, b, w already on fmt's grid."""
    bits = np.atleast_2d(bits).astype(np.float64)
    theta = bits @ w.T + b[None, :]
    xr, xi = _round(theta.real, fmt), _round(theta.imag, fmt)
    lc = re_logcosh(xr, xi)
    lcq = lc if fmt == "f32" else _round(lc, fmt)
    h = lcq.astype(np.float32).sum(axis=1, dtype=np.float32).astype(np.float64)
    vis = (bits @ a.real).astype(np.float32).astype(np.float64)
    lp = 2.0 * (vis + h).astype(np.float32).astype(np.float64)
    ulp = {"f16": 2.0**-10, "bf16": 2.0**-7, "f32": 2.0**-22}[fmt]
    tol = 2.0 * (ulp * np.abs(lc).sum(axis=1) + 2e-6 * lc.shape[1] + 1e-6 * np.abs(lp))
    return lp, tol
