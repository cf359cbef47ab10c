"""Closed-form MH bias bounds logged by the training loop (API names of the
reference bounds.py: pinsker_tv_bound, expected_exp_abs_increment,
theorem3_gaussian_bound; the arithmetic here is this package's own).

For Gaussian log-density noise of std sigma the proposal increments of the
perturbation, eps = delta(y) - delta(x), are N(mu, 2 sigma^2), and the paper's
Theorem 3 bounds the stationary TV distance by (1 - E[e^{-|eps|}]) / (1 - r).
Host scalar math on logged statistics, not the hot path.
"""
from __future__ import annotations

import math

from scipy.special import erfcx, log_ndtr


def pinsker_tv_bound(sigma: float) -> float:
    """KL / Pinsker bound TV <= sigma / 2 for Gaussian log-density noise."""
    if sigma < 0:
        raise ValueError(f"sigma must be non-negative, got {sigma}")
    return sigma / 2.0


def expected_exp_abs_increment(sigma: float, mu: float = 0.0) -> float:
    """E[exp(-|eps|)] for eps ~ N(mu, s^2), s^2 = 2 sigma^2.

    Splitting at 0, each half is a shifted Gaussian tail:
      E = e^{s^2/2 - mu} Phi((mu - s^2)/s) + e^{s^2/2 + mu} Phi(-(mu + s^2)/s),
    evaluated in log space (log_ndtr) so neither factor over- or underflows.
    For mu = 0 it is erfcx(sigma)."""
    if sigma < 0:
        raise ValueError(f"sigma must be non-negative, got {sigma}")
    if sigma == 0.0:
        return math.exp(-abs(mu))
    if mu == 0.0:
        return float(erfcx(sigma))
    s2 = 2.0 * sigma * sigma
    s = math.sqrt(s2)
    upper = 0.5 * s2 - mu + float(log_ndtr((mu - s2) / s))
    lower = 0.5 * s2 + mu + float(log_ndtr(-(mu + s2) / s))
    return math.exp(upper) + math.exp(lower)


def theorem3_gaussian_bound(sigma: float, mu: float = 0.0, r: float = 0.0) -> float:
    """The paper's Theorem 3 TV bound (1 - E[e^{-|eps|}]) / (1 - r), r the
    chain's contraction constant."""
    if not (0.0 <= r < 1.0):
        raise ValueError(f"contraction constant must lie in [0, 1), got {r}")
    if sigma < 0:
        raise ValueError(f"sigma must be non-negative, got {sigma}")
    if sigma == 0.0:
        if mu != 0.0:
            raise ValueError("a zero-variance increment with non-zero mean is outside the bound")
        return 0.0
    return (1.0 - expected_exp_abs_increment(sigma, mu)) / (1.0 - r)
