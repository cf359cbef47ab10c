"""ctypes wrapper of the plain-C oracle ``oracle/c/oracle_port.c`` — test infrastructure only.

Every function mirrors one reference entry point (file:line in the C source).
Format codes: 0=f64, 1=f32, 2=f16, 3=bf16 (``precision.py:64-67`` of the reference).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "liboracle_port.so")
_lib = None

FMT_CODES = {"f64": 0, "f32": 1, "f16": 2, "bf16": 3}

_dp = ctypes.POINTER(ctypes.c_double)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_i64p = ctypes.POINTER(ctypes.c_int64)


class _Model(ctypes.Structure):
    _fields_ = [
        ("N", ctypes.c_int), ("M", ctypes.c_int), ("fmt", ctypes.c_int),
        ("a_re", _dp), ("a_im", _dp), ("b_re", _dp), ("b_im", _dp), ("w_re", _dp), ("w_im", _dp),
    ]


def build():
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_mix64.restype = ctypes.c_uint64
        L.orc_mix64.argtypes = [ctypes.c_uint64]
        L.orc_stream_uniform.restype = ctypes.c_double
        L.orc_stream_uniform.argtypes = [ctypes.c_uint64] * 3
        L.orc_stream_uniforms.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64,
                                          ctypes.c_int64, ctypes.c_int64, _dp]
        L.orc_quantize_fmt.restype = ctypes.c_double
        L.orc_quantize_fmt.argtypes = [ctypes.c_double, ctypes.c_int]
        L.orc_quantize_array.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, _dp]
        L.orc_rounded_forward.argtypes = [_u8p, ctypes.c_int64, ctypes.c_int, ctypes.c_int] + [_dp] * 6 + [
            ctypes.c_int, _dp, _dp, _dp, ctypes.c_int]
        L.orc_rounded_log_prob.argtypes = [_u8p, ctypes.c_int64, ctypes.c_int, ctypes.c_int] + [_dp] * 5 + [
            ctypes.c_int, _dp, ctypes.c_int]
        L.orc_f64_forward.argtypes = [_u8p, ctypes.c_int64, ctypes.c_int, ctypes.c_int] + [_dp] * 6 + [
            _dp, _dp, _dp, ctypes.c_int]
        L.orc_chains_init.restype = ctypes.c_int64
        L.orc_chains_init.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int,
                                      ctypes.c_int, ctypes.c_int, _u8p]
        L.orc_log_probs.argtypes = [ctypes.POINTER(_Model), _u8p, ctypes.c_int64, _dp, ctypes.c_int]
        L.orc_chains_step.argtypes = [ctypes.POINTER(_Model), ctypes.c_uint64, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int, _u8p, _dp, _i64p, ctypes.c_int64,
                                      ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                      _u8p, ctypes.c_int]
        L.orc_local_energies.restype = ctypes.c_int
        L.orc_local_energies.argtypes = [ctypes.POINTER(_Model), ctypes.c_int, _i64p, ctypes.c_int,
                                         ctypes.c_double, ctypes.c_double, _u8p, ctypes.c_int64,
                                         _dp, _dp, ctypes.c_int]
        _lib = L
    return _lib


def _threads(n):
    return int(n) if n else len(os.sched_getaffinity(0))


def _d(a):
    return a.ctypes.data_as(_dp)


def _u8(a):
    return a.ctypes.data_as(_u8p)


class Params:
    """Split re/im float64 copies of complex (a, b, w) arrays (w is (M, N) row-major)."""

    def __init__(self, a, b, w):
        a = np.asarray(a, dtype=np.complex128)
        b = np.asarray(b, dtype=np.complex128)
        w = np.asarray(w, dtype=np.complex128)
        self.N, self.M = a.size, b.size
        self.arrays = [np.ascontiguousarray(v) for v in (a.real, a.imag, b.real, b.imag, w.real, w.imag)]

    def model(self, fmt):
        a_re, a_im, b_re, b_im, w_re, w_im = self.arrays
        return _Model(self.N, self.M, FMT_CODES[fmt] if isinstance(fmt, str) else int(fmt),
                      _d(a_re), _d(a_im), _d(b_re), _d(b_im), _d(w_re), _d(w_im))


def stream_uniforms(key, n_chains, n_draws, chain0=0, t0=0):
    out = np.empty((n_draws, n_chains))
    lib().orc_stream_uniforms(int(key), n_chains, chain0, t0, n_draws, _d(out))
    return out


def quantize(v, fmt):
    return lib().orc_quantize_fmt(float(v), FMT_CODES[fmt])


def quantize_array(values, fmt):
    """Elementwise RNE rounding to fmt (f64 arrays)."""
    v = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty_like(v)
    lib().orc_quantize_array(_d(v), v.size, FMT_CODES[fmt], _d(out))
    return out


def random_parameters(n_visible, alpha, key, scale=0.01):
    """rbm.random_parameters (rbm.py:78-88): Re and Im i.i.d. N(0, scale^2) from the
    counter-based Gaussian field, order [a | b | W row-major] (re block, then im
    block).  Returns complex (a, b, w) with w of shape (M, N)."""
    from fractions import Fraction

    from oracle.rng import gaussian_field

    m = Fraction(alpha) * n_visible
    if m.denominator != 1 or m <= 0:
        raise ValueError("alpha*N must be a positive integer")
    m = int(m)
    count = n_visible + m + m * n_visible
    draws = scale * gaussian_field(key, np.arange(2 * count), 1.0)
    z = draws[:count] + 1j * draws[count:]
    return z[:n_visible], z[n_visible:n_visible + m], z[n_visible + m:].reshape(m, n_visible)


def round_parameters(a, b, w, fmt):
    """rbm.round_parameters (rbm.py:91-101): Re and Im rounded RNE to fmt."""
    if fmt == "f64":
        return a, b, w
    q = lambda z: quantize_array(z.real, fmt) + 1j * quantize_array(z.imag, fmt)  # noqa: E731
    return q(a), q(b), q(w)


def rounded_forward(params: Params, bits, fmt, nthreads=None):
    """_kernels.rounded_forward: (lp, re, im) in per-operation rounding."""
    bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
    B = bits.shape[0]
    lp, re, im = np.empty(B), np.empty(B), np.empty(B)
    a_re, a_im, b_re, b_im, w_re, w_im = params.arrays
    lib().orc_rounded_forward(_u8(bits), B, params.N, params.M, _d(a_re), _d(a_im), _d(b_re), _d(b_im),
                              _d(w_re), _d(w_im), FMT_CODES[fmt], _d(lp), _d(re), _d(im), _threads(nthreads))
    return lp, re, im


def rounded_log_prob(params: Params, bits, fmt, nthreads=None):
    bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
    lp = np.empty(bits.shape[0])
    a_re, _, b_re, b_im, w_re, w_im = params.arrays
    lib().orc_rounded_log_prob(_u8(bits), bits.shape[0], params.N, params.M, _d(a_re), _d(b_re), _d(b_im),
                               _d(w_re), _d(w_im), FMT_CODES[fmt], _d(lp), _threads(nthreads))
    return lp


def f64_forward(params: Params, bits, nthreads=None):
    bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
    B = bits.shape[0]
    lp, re, im = np.empty(B), np.empty(B), np.empty(B)
    a_re, a_im, b_re, b_im, w_re, w_im = params.arrays
    lib().orc_f64_forward(_u8(bits), B, params.N, params.M, _d(a_re), _d(a_im), _d(b_re), _d(b_im),
                          _d(w_re), _d(w_im), _d(lp), _d(re), _d(im), _threads(nthreads))
    return lp, re, im


class PortEnsemble:
    """ChainEnsemble (sampler.py:48-167) on the C port: per-operation evaluator
    for f32/f16/bf16, sequential-sum f64 forward for f64."""

    def __init__(self, n_chains, n_sites, proposal, sector_weight, params: Params, fmt, key,
                 chain0=0, nthreads=None):
        self.n_chains, self.n_sites = int(n_chains), int(n_sites)
        self.kind = 0 if proposal == "flip" else 1
        self.params, self.fmt, self.key, self.chain0 = params, fmt, int(key), int(chain0)
        self.nthreads = _threads(nthreads)
        self._model = params.model(fmt)
        self.bits = np.empty((self.n_chains, self.n_sites), dtype=np.uint8)
        weight = self.n_sites // 2 if sector_weight is None else int(sector_weight)
        self.t_draw = lib().orc_chains_init(self.key, self.n_chains, self.chain0, self.n_sites, self.kind,
                                            weight, _u8(self.bits))
        self.logp = np.empty(self.n_chains)
        lib().orc_log_probs(ctypes.byref(self._model), _u8(self.bits), self.n_chains, _d(self.logp),
                            self.nthreads)
        self.acc = np.zeros(self.n_chains, dtype=np.int64)
        self.proposed = 0

    def set_params(self, params: Params, fmt=None):
        """ChainEnsemble.set_evaluator (sampler.py:90-93): new target, cached log p
        refreshed with one batched evaluation of every chain."""
        self.params = params
        self.fmt = fmt if fmt is not None else self.fmt
        self._model = params.model(self.fmt)
        lib().orc_log_probs(ctypes.byref(self._model), _u8(self.bits), self.n_chains, _d(self.logp),
                            self.nthreads)

    @property
    def accepted(self):
        return int(self.acc.sum())

    def reset_counters(self):
        self.acc[:] = 0
        self.proposed = 0

    def run_steps(self, n_steps, thin=0, base=0, extra=0, samples=None):
        lib().orc_chains_step(ctypes.byref(self._model), self.key, self.n_chains, self.chain0, self.kind,
                              _u8(self.bits), _d(self.logp), self.acc.ctypes.data_as(_i64p), self.t_draw,
                              int(n_steps), int(thin), int(base), int(extra),
                              _u8(samples) if samples is not None else None, self.nthreads)
        self.t_draw += 2 * int(n_steps)
        self.proposed += self.n_chains * int(n_steps)

    def collect(self, n_samples, thin_steps=1):
        base, extra = divmod(int(n_samples), self.n_chains)
        rounds = base + (1 if extra else 0)
        samples = np.zeros((n_samples, self.n_sites), dtype=np.uint8)
        self.run_steps(rounds * thin_steps, thin_steps, base, extra, samples)
        return samples


def local_energies(params: Params, ham, bonds, J, h, bits, nthreads=None):
    """vmc.local_energies with the f64 forward (ham: 'tfim' or 'heisenberg')."""
    bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
    bonds = np.ascontiguousarray(np.asarray(bonds, dtype=np.int64).reshape(-1, 2))
    B = bits.shape[0]
    er, ei = np.empty(B), np.empty(B)
    model = params.model("f64")
    bad = lib().orc_local_energies(ctypes.byref(model), 0 if ham == "tfim" else 1,
                                   bonds.ctypes.data_as(_i64p), bonds.shape[0], float(J), float(h),
                                   _u8(bits), B, _d(er), _d(ei), _threads(nthreads))
    if bad:
        raise FloatingPointError("non-finite local energy (oracle)")
    return er + 1j * ei
