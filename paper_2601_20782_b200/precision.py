"""Number formats of the two-copy scheme and the rounding modes of the
evaluators.  API names follow the reference (`precision.py:23-169`:
FloatFormat, BF16/F16/F32/F64, parse_format, RoundingMode, make_rounder,
round_to_format); the implementation is this package's own.

Formats are described by (exponent bits, explicit significand bits).  Host
rounding is only used to build the parameter snapshot (rbm.round_parameters);
every per-sample operation runs in the CUDA library, where the reduced formats
are native (`add.rn.{f16,bf16,f32}`, `cvt.rn.*`).

Rounding modes: STORAGE_ONLY and PER_OPERATION as in the reference, plus
NATIVE, the fused-sweep arithmetic of this package: theta is
kept exact on chip and rounded once to the format, each hidden unit's
Re log cosh is evaluated in f32 and rounded to the format, the hidden sum is
accumulated in f32.
"""
from __future__ import annotations

import enum
import re
from dataclasses import dataclass

import numpy as np

_DEVICE_CODES = {"f64": 0, "f32": 1, "f16": 2, "bf16": 3}  # MPV_FMT_* (include/mpvmc_b200.h)


@dataclass(frozen=True)
class FloatFormat:
    """Binary floating-point format: `exponent_bits` and `significand_bits`
    (without the implicit leading one); subnormals optional."""

    name: str
    exponent_bits: int
    significand_bits: int
    supports_subnormals: bool = True

    def __post_init__(self):
        if not (2 <= self.exponent_bits <= 11 and 1 <= self.significand_bits <= 52):
            raise ValueError(f"format {self.name!r}: exponent bits must lie in [2, 11] and significand bits "
                             "in [1, 52] (float64 is the widest emulated format)")

    @property
    def bias(self) -> int:
        return 2 ** (self.exponent_bits - 1) - 1

    @property
    def max_exponent(self) -> int:
        return self.bias

    @property
    def min_exponent(self) -> int:
        return 1 - self.bias

    @property
    def max_finite(self) -> float:
        return float(np.ldexp(2.0 - np.ldexp(1.0, -self.significand_bits), self.max_exponent))

    @property
    def min_normal(self) -> float:
        return float(np.ldexp(1.0, self.min_exponent))

    @property
    def unit_roundoff(self) -> float:
        return float(np.ldexp(1.0, -self.significand_bits - 1))

    @property
    def code(self) -> int:
        """MPV_FMT_* code of the C ABI."""
        if self.name not in _DEVICE_CODES:
            raise ValueError(f"no device kernels for format {self.name!r}")
        return _DEVICE_CODES[self.name]


F64 = FloatFormat("f64", 11, 52)
F32 = FloatFormat("f32", 8, 23)
F16 = FloatFormat("f16", 5, 10)
BF16 = FloatFormat("bf16", 8, 7)
FORMATS = {f.name: f for f in (F64, F32, F16, BF16)}
FORMAT_CODES = dict(_DEVICE_CODES)

_EM_NAME = re.compile(r"e(?P<e>\d+)m(?P<m>\d+)")


def parse_format(name: str) -> FloatFormat:
    """A named format (f64 / f32 / f16 / bf16) or a custom `e<E>m<M>`."""
    fmt = FORMATS.get(name)
    if fmt is not None:
        return fmt
    m = _EM_NAME.fullmatch(name)
    if m is None:
        raise ValueError(f"{name!r} is neither f64/f32/f16/bf16 nor e<E>m<M>")
    return FloatFormat(name, int(m["e"]), int(m["m"]))


class RoundingMode(enum.Enum):
    """Where results are rounded to the format."""

    STORAGE_ONLY = "storage_only"    # parameters stored in fmt, arithmetic in f64
    PER_OPERATION = "per_operation"  # every add rounded (the reference's emulation)
    NATIVE = "native"                # the B200 fused-sweep arithmetic

    @property
    def code(self) -> int:
        return (RoundingMode.NATIVE, RoundingMode.PER_OPERATION, RoundingMode.STORAGE_ONLY).index(self)


def parse_rounding_mode(name: str) -> RoundingMode:
    try:
        return RoundingMode(name)
    except ValueError:
        raise ValueError(f"rounding mode must be one of {[m.value for m in RoundingMode]}, got {name!r}") from None


def _rne_generic(x: np.ndarray, fmt: FloatFormat) -> np.ndarray:
    """Round-to-nearest-even onto fmt's grid by bit arithmetic on the float64
    pattern: add half an ulp of the target (minus one when the kept lsb is 0),
    clear the dropped bits; values below fmt's normal range are rounded on the
    fixed subnormal grid (or flushed), overflow goes to +-inf."""
    x = np.asarray(x, dtype=np.float64)
    out = np.array(x, dtype=np.float64, copy=True)
    finite = np.isfinite(x)
    drop = 52 - fmt.significand_bits
    if drop > 0:
        u = x.view(np.uint64)
        half = np.uint64(1 << (drop - 1))
        lsb = (u >> np.uint64(drop)) & np.uint64(1)
        mask = ~np.uint64((1 << drop) - 1)
        r = ((u + half - np.uint64(1) + lsb) & mask).view(np.float64)
        out = np.where(finite, r, x)
    tiny = np.abs(x) < fmt.min_normal
    if np.any(tiny & finite):
        step = np.ldexp(1.0, fmt.min_exponent - fmt.significand_bits)  # subnormal spacing
        xt = np.where(tiny & finite, x, 0.0)
        sub = np.rint(xt / step) * step  # exact scaling, numpy rint is half-to-even
        if not fmt.supports_subnormals:
            sub = np.where(np.abs(sub) < fmt.min_normal, 0.0 * xt, sub)
        out = np.where(tiny & finite, sub, out)
    with np.errstate(invalid="ignore"):
        big = np.abs(out) > fmt.max_finite
    return np.where(big & finite, np.copysign(np.inf, x), out)


def make_rounder(fmt: FloatFormat):
    """Vectorised RNE rounding onto fmt (float64 in, float64 out)."""
    if fmt.name == "f64":
        return lambda a: np.asarray(a, dtype=np.float64)
    native = {"f32": np.float32, "f16": np.float16}.get(fmt.name)
    if native is not None and fmt.supports_subnormals:
        return lambda a: np.asarray(a, dtype=np.float64).astype(native).astype(np.float64)
    return lambda a: _rne_generic(a, fmt)


def round_to_format(value, fmt: FloatFormat):
    """Scalar or array rounding onto fmt."""
    arr = np.asarray(value, dtype=np.float64)
    with np.errstate(over="ignore"):
        out = make_rounder(fmt)(arr)
    return float(out) if arr.ndim == 0 else out
