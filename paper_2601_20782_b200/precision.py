"""Floating-point formats and rounding modes (mirror of the reference's
precision.py:23-169; same names and semantics).

Adds one rounding mode, ``NATIVE``: the B200 fused-sweep arithmetic.  The
hidden pre-activation theta(x) = b + W x is kept exact (on-chip accumulators,
see DESIGN.md §3) and rounded ONCE to the format, each hidden unit's
Re log cosh is evaluated in f32 from that rounded value and rounded to the
format, and the hidden sum is accumulated in f32.  log p_fmt(x) is therefore a
fixed function of x (path independent), which is what the paper's
perturbed-target bounds assume.

Host-side rounding here is only used for the two-copy parameter snapshot
(rbm.round_parameters, reference rbm.py:91-101); all per-sample arithmetic runs
in the CUDA library.
"""
from __future__ import annotations

import enum
import re
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class FloatFormat:
    """An (exponent bits, significand bits) pair; significand_bits excludes the
    implicit leading 1 (reference precision.py:23-61)."""

    name: str
    exponent_bits: int
    significand_bits: int
    supports_subnormals: bool = True

    def __post_init__(self):
        if self.exponent_bits < 2 or self.significand_bits < 1:
            raise ValueError("need >= 2 exponent bits and >= 1 significand bit")
        if self.exponent_bits > 11 or self.significand_bits > 52:
            raise ValueError("formats wider than float64 cannot be emulated")

    @property
    def bias(self) -> int:
        return (1 << (self.exponent_bits - 1)) - 1

    @property
    def max_exponent(self) -> int:
        return self.bias

    @property
    def min_exponent(self) -> int:
        return 1 - self.bias

    @property
    def max_finite(self) -> float:
        return (2.0 - 2.0 ** -self.significand_bits) * 2.0 ** self.max_exponent

    @property
    def min_normal(self) -> float:
        return 2.0 ** self.min_exponent

    @property
    def unit_roundoff(self) -> float:
        return 2.0 ** -(self.significand_bits + 1)

    @property
    def code(self) -> int:
        """Format code of the C-ABI (include/mpvmc_b200.h, MPV_FMT_*)."""
        try:
            return FORMAT_CODES[self.name]
        except KeyError:
            raise ValueError(f"format {self.name!r} has no device implementation") from None


BF16 = FloatFormat("bf16", 8, 7)
F16 = FloatFormat("f16", 5, 10)
F32 = FloatFormat("f32", 8, 23)
F64 = FloatFormat("f64", 11, 52)

FORMATS = {fmt.name: fmt for fmt in (BF16, F16, F32, F64)}
FORMAT_CODES = {"f64": 0, "f32": 1, "f16": 2, "bf16": 3}
_CUSTOM_RE = re.compile(r"^e(\d+)m(\d+)$")


def parse_format(name: str) -> FloatFormat:
    """Resolve a format name: f64/f32/f16/bf16 or custom e<E>m<M> (precision.py:74-81)."""
    if name in FORMATS:
        return FORMATS[name]
    match = _CUSTOM_RE.match(name)
    if match:
        return FloatFormat(name, int(match.group(1)), int(match.group(2)))
    raise ValueError(f"unknown float format {name!r}")


class RoundingMode(enum.Enum):
    """Where rounding is applied (precision.py:158-169) plus the device NATIVE mode."""

    STORAGE_ONLY = "storage_only"
    PER_OPERATION = "per_operation"
    NATIVE = "native"

    @property
    def code(self) -> int:
        return {"native": 0, "per_operation": 1, "storage_only": 2}[self.value]


def parse_rounding_mode(name: str) -> RoundingMode:
    for mode in RoundingMode:
        if mode.value == name:
            return mode
    raise ValueError(f"unknown rounding mode {name!r}")


def _quantize(values: np.ndarray, fmt: FloatFormat) -> np.ndarray:
    """Round-to-nearest-even onto fmt's grid; overflow -> +-inf; subnormals kept
    unless the format flushes them (same contract as precision.py:89-104)."""
    with np.errstate(all="ignore"):
        _, exponents = np.frexp(values)
        eu = np.maximum(exponents - 1, fmt.min_exponent)
        quantum = np.ldexp(1.0, eu - fmt.significand_bits)
        rounded = np.rint(values / quantum) * quantum
        if not fmt.supports_subnormals:
            rounded = np.where(np.abs(rounded) < fmt.min_normal, 0.0 * rounded, rounded)
        return np.where(np.abs(rounded) > fmt.max_finite, np.copysign(np.inf, rounded), rounded)


def make_rounder(fmt: FloatFormat):
    """Array rounding callable (precision.py:107-132)."""
    if fmt.name == "f64":
        return lambda a: np.asarray(a, dtype=np.float64)
    if fmt.name == "f32":
        return lambda a: np.asarray(a, dtype=np.float64).astype(np.float32).astype(np.float64)
    if fmt.name == "f16":
        return lambda a: np.asarray(a, dtype=np.float64).astype(np.float16).astype(np.float64)
    return lambda a: _quantize(np.asarray(a, dtype=np.float64), fmt)


def round_to_format(value, fmt: FloatFormat):
    arr = np.asarray(value, dtype=np.float64)
    with np.errstate(over="ignore"):
        out = make_rounder(fmt)(arr)
    if np.isscalar(value) or arr.ndim == 0:
        return float(out)
    return out
