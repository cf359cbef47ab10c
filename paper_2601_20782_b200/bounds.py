"""Closed-form MH bias bounds logged by the training loop (mirror of the
reference bounds.py:28-47, 78-83, 192-229): Pinsker TV <= sigma/2 and the
Gaussian-increment Theorem 3.  Host scalar math (logging, not the hot path)."""
from __future__ import annotations

import math

from scipy.special import erfcx as _erfcx


def pinsker_tv_bound(sigma: float) -> float:
    """TV <= sigma/2 for Gaussian log-density noise of std sigma (bounds.py:78-83)."""
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    return 0.5 * sigma


def expected_exp_abs_increment(sigma: float, mu: float = 0.0) -> float:
    """E[e^-|eps|] for eps ~ N(mu, 2 sigma^2) via the scaled erfc (bounds.py:192-214)."""
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    if sigma == 0.0:
        return math.exp(-abs(mu))
    shift = mu / (2.0 * sigma)

    def piece(t, reflected_exponent):
        if t > -25.0:
            return math.exp(-shift * shift) * float(_erfcx(t))
        return 2.0 * math.exp(reflected_exponent) - math.exp(-shift * shift) * float(_erfcx(-t))

    return 0.5 * (piece(sigma - shift, sigma * sigma - mu) + piece(sigma + shift, sigma * sigma + mu))


def theorem3_gaussian_bound(sigma: float, mu: float = 0.0, r: float = 0.0) -> float:
    """(1 - E[e^-|eps|]) / (1 - r) (bounds.py:217-229)."""
    if not 0.0 <= r < 1.0:
        raise ValueError("contraction constant r must be in [0, 1)")
    if sigma < 0:
        raise ValueError("sigma must be >= 0")
    if sigma == 0.0:
        if mu != 0.0:
            raise ValueError("sigma = 0 with mu != 0 is outside the bound's domain")
        return 0.0
    return (1.0 - expected_exp_abs_increment(sigma, mu)) / (1.0 - r)
