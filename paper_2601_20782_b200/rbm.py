"""RBM neural quantum state on the B200: parameters (host, f64 master copy),
the reduced-precision snapshot in kernel layout (device), and the evaluator
objects the sampler and the local energies consume.

Mirrors the reference rbm.py API: ``RbmParameters`` (rbm.py:27-75),
``random_parameters`` (:78-88), ``round_parameters`` (:91-101),
``save_parameters``/``load_parameters`` (:104-127), ``log_prob_evaluator``
(:361-405), ``log_psi_evaluator`` (:419-425), ``log_prob_batch``/``log_psi_batch``
(:254-296), ``grad_log_psi_batch`` (:307-325).  Evaluation always runs in the
CUDA library; the evaluators are device objects that ``ChainEnsemble``
recognises and fuses, and they stay callable on uint8 numpy rows (host round
trip) so reference callers keep working.
"""
from __future__ import annotations

import ctypes
import json
import math
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _native as nat
from .errors import EvaluationFailureError
from .lattice import pack_bits
from .precision import F64, FloatFormat, RoundingMode, make_rounder
from .rng import derive_key, gaussian_field


def _as_complex(name: str, value, ndim: int) -> np.ndarray:
    arr = np.asarray(value, dtype=np.complex128)
    if arr.ndim != ndim:
        raise ValueError(f"{name} must be {ndim}-dimensional, got shape {arr.shape}")
    if not np.isfinite(arr.view(np.float64)).all():
        raise ValueError(f"{name} has non-finite entries")
    return arr


@dataclass(frozen=True)
class RbmParameters:
    """Complex RBM parameters: visible biases a [N], hidden biases b [M], weights
    w [M, N] (the reference's RbmParameters fields and flat order a, b, W)."""

    a: np.ndarray
    b: np.ndarray
    w: np.ndarray

    def __post_init__(self):
        a, b, w = _as_complex("a", self.a, 1), _as_complex("b", self.b, 1), _as_complex("w", self.w, 2)
        if w.shape != (b.size, a.size):
            raise ValueError(f"w has shape {w.shape}, expected (len(b), len(a)) = ({b.size}, {a.size})")
        for name, arr in (("a", a), ("b", b), ("w", w)):
            object.__setattr__(self, name, arr)

    n_visible = property(lambda self: self.a.size)
    n_hidden = property(lambda self: self.b.size)
    alpha_density = property(lambda self: Fraction(self.n_hidden, self.n_visible))
    n_params = property(lambda self: self.a.size + self.b.size + self.w.size)

    def flatten(self) -> np.ndarray:
        """theta = [a | b | W row-major]."""
        return np.concatenate((self.a, self.b, self.w.ravel()))

    @classmethod
    def from_flat(cls, theta, n_visible: int, n_hidden: int) -> "RbmParameters":
        theta = np.asarray(theta, dtype=np.complex128)
        cut = np.cumsum([n_visible, n_hidden])
        a, b, w = np.split(theta, cut)
        return cls(a, b, w.reshape(n_hidden, n_visible))


def random_parameters(n_visible: int, alpha, key, scale: float = 0.01) -> RbmParameters:
    """Gaussian initialisation from the counter-based field (rng.gaussian_field):
    counters 0..P-1 give the real parts and P..2P-1 the imaginary parts of
    theta = [a | b | W], each N(0, scale^2) (the reference's draw order)."""
    m = Fraction(alpha) * n_visible
    if m.denominator != 1 or m <= 0:
        raise ValueError(f"alpha * n_visible = {m} is not a positive integer")
    m = int(m)
    total = n_visible + m + m * n_visible
    z = scale * gaussian_field(key, np.arange(2 * total), 1.0)
    return RbmParameters.from_flat(z[:total] + 1j * z[total:], n_visible, m)


def round_parameters(params: RbmParameters, fmt: FloatFormat) -> RbmParameters:
    """The two-copy snapshot: real and imaginary parts rounded to fmt (RNE)."""
    if fmt.name == "f64":
        return params
    rnd = make_rounder(fmt)
    with np.errstate(over="ignore"):
        parts = [rnd(arr.real) + 1j * rnd(arr.imag) for arr in (params.a, params.b, params.w)]
    return RbmParameters(*parts)


_PARAMS_FORMAT = "rbm-params-v1"


def save_parameters(params: RbmParameters, path):
    """JSON file in the reference's rbm-params-v1 layout: every complex number
    as a [re, im] pair."""
    pairs = lambda z: np.stack([z.real, z.imag], axis=-1).tolist()  # noqa: E731
    doc = {"format": _PARAMS_FORMAT, "n_visible": params.n_visible, "n_hidden": params.n_hidden,
           "a": pairs(params.a), "b": pairs(params.b), "w": pairs(params.w)}
    with open(path, "w") as fh:
        json.dump(doc, fh)


def load_parameters(path) -> RbmParameters:
    with open(path) as fh:
        doc = json.load(fh)
    if doc.get("format") != _PARAMS_FORMAT:
        raise ValueError(f"{path}: not an {_PARAMS_FORMAT} file")
    cplx = lambda v: (lambda arr: arr[..., 0] + 1j * arr[..., 1])(np.asarray(v, dtype=np.float64))  # noqa: E731
    return RbmParameters(cplx(doc["a"]), cplx(doc["b"]), cplx(doc["w"]))


# ---------------------------------------------------------------------------
# Exact-theta planner
# ---------------------------------------------------------------------------

def finest_quantum(values: np.ndarray) -> float:
    """Largest power of two dividing every nonzero finite value (1.0 if none)."""
    v = np.abs(np.asarray(values, dtype=np.float64).ravel())
    v = v[(v != 0) & np.isfinite(v)]
    if v.size == 0:
        return 1.0
    m, e = np.frexp(v)
    mi = (m * 2.0**53).astype(np.int64)
    tz = np.log2((mi & -mi).astype(np.float64)).astype(np.int64)
    return float(np.ldexp(1.0, int((e.astype(np.int64) - 53 + tz).min())))


@dataclass(frozen=True)
class ExactPlan:
    """Which on-chip accumulator keeps theta = b + W x exact for a snapshot.

    All partial sums of the snapshot's values are multiples of ``quantum`` and
    bounded by ``bound``; f32 holds every multiple of q up to 2^24 q exactly.
    X1: one f32 per component (bound <= 2^24 q).  XI: one int32 per component
    counting multiples of q (bound < 2^30 q, q >= 2^-100).  X2: theta = hi + lo with hi on the
    grid ``split`` (|hi| <= 2^24 split) and |lo| <= (N+1) split/2 <= 2^24 q.
    F64: otherwise (f64 accumulators, converted per unit)."""

    variant: int
    quantum: float
    bound: float
    split: float


def plan_from_bounds(q: float, bound_re: float, bound_im: float, bound_a: float, n_visible: int,
                     allow_xi: bool = True) -> ExactPlan:
    """The planner's decision from the snapshot's quantum and bounds (XI, the
    integer accumulators, exists for the f16/bf16 kernels only: allow_xi)."""
    bound = max(bound_re, bound_im, bound_a)
    n_terms = n_visible + 1
    split = 2.0 ** math.floor(math.log2(2.0**25 * q / n_terms))
    if not (split >= q and bound + n_terms * split / 2 <= 2.0**24 * split):
        split = 0.0  # X2 not exact
    if bound <= 2.0**24 * q:
        return ExactPlan(nat.ACC_X1, q, bound, split)
    if allow_xi and bound < 2.0**30 * q and q >= 2.0**-100:  # q applied in f32 (bf16: exact above 2^-100)
        return ExactPlan(nat.ACC_XI, q, bound, split)
    if split > 0.0:
        return ExactPlan(nat.ACC_X2, q, bound, split)
    return ExactPlan(nat.ACC_F64, q, bound, 0.0)


def plan_exact(snap: RbmParameters, allow_xi: bool = True) -> ExactPlan:
    """Host planner on a rounded snapshot (the device computes the same four
    numbers in mpv_snapshot_round)."""
    a, b, w = snap.a, snap.b, snap.w
    vals = np.concatenate([a.real, b.real, b.imag, w.real.ravel(), w.imag.ravel()])
    return plan_from_bounds(finest_quantum(vals), float(np.max(np.abs(b.real) + np.abs(w.real).sum(axis=1))),
                            float(np.max(np.abs(b.imag) + np.abs(w.imag).sum(axis=1))),
                            float(np.abs(a.real).sum()), snap.n_visible, allow_xi)


# ---------------------------------------------------------------------------
# Device snapshot (kernel layout)
# ---------------------------------------------------------------------------

class DeviceSnapshot:
    """Parameters of one evaluator in kernel layout, resident on the device
    (the device counterpart of rbm.py:161-200 _PreparedRounded).

    Built on the device: one upload of the f64 master parameters,
    mpv_snapshot_round (RNE rounding to fmt + the planner's quantum/bounds),
    the host planner's decision on those four numbers, then mpv_snapshot_fill
    writes the table in the chosen layout."""

    def __init__(self, params: RbmParameters, fmt: FloatFormat, mode: RoundingMode, device=None,
                 variant: int | None = None):
        import torch

        nat.require_cuda()
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.fmt, self.mode = fmt, mode
        f64arith = fmt.name == "f64" or mode is RoundingMode.STORAGE_ONLY
        N, M = params.n_visible, params.n_hidden
        self.n_visible, self.n_hidden = N, M
        stream = nat.stream_handle(self.device)
        # [a | b | w_t] as interleaved (re, im) f64, one pinned upload
        host = torch.empty(2 * (N + M + N * M), dtype=torch.float64, pin_memory=True)
        hv = host.numpy().view(np.complex128)
        hv[:N], hv[N:N + M] = params.a, params.b
        hv[N + M:].reshape(N, M)[:] = params.w.T
        src = host.to(self.device, non_blocking=True)
        self._rounded = torch.empty_like(src)
        plan_dev = torch.empty(8, dtype=torch.float64, device=self.device)
        nat.call("mpv_snapshot_round", N, M, fmt.code, src.data_ptr(), self._rounded.data_ptr(), plan_dev.data_ptr(),
                 stream)
        split = 0.0
        quantum = 0.0
        cluster = 1
        if mode is RoundingMode.PER_OPERATION and not f64arith:
            G, U, Mpad = 1, M, M
            variant = nat.ACC_X1
        else:
            if f64arith:
                variant = nat.ACC_F64
            else:
                pq = plan_dev.cpu().numpy()
                self.plan = plan_from_bounds(float(pq[0]), float(pq[1]), float(pq[2]), float(pq[3]), N,
                                             allow_xi=fmt.name in ("f16", "bf16"))
                if variant is None:
                    variant = self.plan.variant
                elif variant == nat.ACC_X1 and self.plan.variant != nat.ACC_X1:
                    raise ValueError("X1 accumulators are not exact for this snapshot")
                elif variant == nat.ACC_X2 and self.plan.split == 0.0:
                    raise ValueError("X2 accumulators are not exact for this snapshot")
                elif variant == nat.ACC_XI and fmt.name not in ("f16", "bf16"):
                    raise ValueError("XI accumulators exist for f16/bf16 snapshots only")
                elif variant == nat.ACC_XI and not (self.plan.bound < 2.0**30 * self.plan.quantum
                                                    and self.plan.quantum >= 2.0**-100):
                    raise ValueError("XI accumulators are not exact for this snapshot")
                split = self.plan.split
                if variant == nat.ACC_XI:
                    quantum = self.plan.quantum
            cluster, G, U = nat.plan_cluster(N, M, fmt.code, mode.code, variant)
            Mpad = cluster * G * U
        self._split, self._quantum = split, quantum
        self._layouts = {}
        self._fill(variant, cluster, G, U, Mpad)

    def _fill(self, variant, cluster, G, U, Mpad):
        """Table, bias and visible terms in the layout (cluster, G, U), filled on
        the device from the rounded parameters."""
        import torch

        N, M, fmt, mode = self.n_visible, self.n_hidden, self.fmt, self.mode
        stream = nat.stream_handle(self.device)
        split, quantum = self._split, self._quantum
        self.variant, self.lanes_per_chain, self.units_per_lane, self.hidden_pad = variant, G, U, Mpad
        self.cluster = cluster
        sizes = (ctypes.c_size_t * 3)()
        nat.call("mpv_snapshot_bytes", N, Mpad, fmt.code, mode.code, variant, cluster, sizes)
        self._table = torch.zeros(int(sizes[0]), dtype=torch.uint8, device=self.device)  # zero padding
        self._bias = torch.zeros(int(sizes[2]), dtype=torch.uint8, device=self.device)
        self._vis_im = torch.empty(N, dtype=torch.float64, device=self.device)
        base = self._table.data_ptr()
        self.struct = nat.Snapshot(N, M, Mpad, fmt.code, mode.code, variant, G, U, cluster,
                                   base, self._bias.data_ptr(), base + int(sizes[1]), self._vis_im.data_ptr(), quantum)
        nat.call("mpv_snapshot_fill", ctypes_byref(self.struct), self._rounded.data_ptr(), split, stream)

    def for_proposal(self, kind: str) -> "DeviceSnapshot":
        """The snapshot in the layout the fused sweep uses for `kind`.  Exchange
        sweeps run one chain per warp (32 lanes per chain, mpv_plan_cluster_ex)
        so a step that swaps equal bits is skipped by the whole warp; the table
        is re-filled once from the same rounded parameters and cached."""
        if kind != "exchange":
            return self
        f64arith = self.fmt.name == "f64" or self.mode is RoundingMode.STORAGE_ONLY
        if self.mode is RoundingMode.PER_OPERATION and not f64arith:
            return self  # the per-operation kernels do not use the lane layout
        if self.cluster > 1:
            return self  # opt-in cluster split (instantiated for G = 8 only)
        cluster, G, U = nat.plan_cluster(self.n_visible, self.n_hidden, self.fmt.code, self.mode.code, self.variant,
                                         32)
        if (cluster, G, U) == (self.cluster, self.lanes_per_chain, self.units_per_lane):
            return self
        key = (cluster, G, U)
        if key not in self._layouts:
            other = object.__new__(DeviceSnapshot)
            other.__dict__.update({k: v for k, v in self.__dict__.items() if k != "_layouts"})
            other._layouts = {}
            other._fill(self.variant, cluster, G, U, cluster * G * U)
            self._layouts[key] = other
        return self._layouts[key]

    @property
    def params(self) -> RbmParameters:
        """The rounded snapshot (ref: rbm.py:91-101), read back from the device."""
        r = self._rounded.cpu().numpy().view(np.complex128)
        N, M = self.n_visible, self.n_hidden
        return RbmParameters(r[:N].copy(), r[N:N + M].copy(), r[N + M:].reshape(N, M).T.copy())

    def scratch(self, n_chains: int):
        """Device scratch for the fused sweep over n_chains (work queue, parked theta)."""
        import torch

        nbytes = nat.load().mpv_sweep_scratch_bytes(ctypes_byref(self.struct), int(n_chains))
        return torch.empty(nbytes, dtype=torch.uint8, device=self.device)

    @property
    def label(self) -> str:
        names = {nat.ACC_X1: "X1", nat.ACC_X2: "X2", nat.ACC_F64: "F64", nat.ACC_XI: "XI"}
        cl = f"C{self.cluster}x" if self.cluster > 1 else ""
        return (f"{self.fmt.name}/{self.mode.value}/{names[self.variant]}/"
                f"{cl}G{self.lanes_per_chain}xU{self.units_per_lane}")


# ---------------------------------------------------------------------------
# Evaluators
# ---------------------------------------------------------------------------

def _status_tensor(device):
    import torch

    return torch.tensor([0, 2**63 - 1], dtype=torch.int64, device=device)


def device_pack(bits, device):
    """uint8 (B, N) host rows -> packed uint32 words on the device (int32 tensor):
    one H2D copy of the rows and the mpv_pack_bits kernel."""
    import torch

    bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
    B, N = bits.shape
    rows = torch.from_numpy(bits)
    if B and not rows.is_pinned():  # stage through pinned memory (DMA instead of a pageable copy)
        rows = torch.empty(rows.shape, dtype=torch.uint8, pin_memory=True).copy_(rows)
    rows = rows.to(device, non_blocking=True)
    packed = torch.empty((B, (N + 31) // 32), dtype=torch.int32, device=device)
    if B:
        nat.call("mpv_pack_bits", rows.data_ptr(), B, N, packed.data_ptr(), nat.stream_handle(device))
    return packed


class LogProbEvaluator:
    """Batch log-probability evaluator ``uint8[B,N] -> float64[B]`` (the
    reference evaluator protocol, sampler.py:49-53) backed by a device snapshot.
    ChainEnsemble fuses it into the MH sweep instead of calling it."""

    def __init__(self, params: RbmParameters, fmt: FloatFormat = F64,
                 mode: RoundingMode = RoundingMode.PER_OPERATION, device=None, variant: int | None = None):
        if fmt.name == "f64":
            mode = RoundingMode.PER_OPERATION  # f64 ignores the mode (rbm.py:364-372)
        self.fmt, self.mode = fmt, mode
        self.master = params
        self.snapshot = DeviceSnapshot(params, fmt, mode, device, variant)
        self.device = self.snapshot.device

    @property
    def n_visible(self):
        return self.snapshot.n_visible

    def for_proposal(self, kind: str) -> "LogProbEvaluator":
        """This evaluator in the lane layout an ensemble with `kind` proposals
        sweeps with (DeviceSnapshot.for_proposal).  With NATIVE arithmetic the
        f32 summation order of the hidden sum follows the layout, so a chain's
        cached log p equals this view's evaluation bit for bit."""
        snap = self.snapshot.for_proposal(kind)
        if snap is self.snapshot:
            return self
        view = object.__new__(type(self))
        view.__dict__.update(self.__dict__)
        view.snapshot = snap
        return view

    def log_prob_packed(self, packed):
        """Device path: packed uint32 [B, words] tensor -> float64 [B] tensor."""
        import torch

        B = packed.shape[0]
        out = torch.empty(B, dtype=torch.float64, device=self.device)
        status = _status_tensor(self.device)
        scratch = self.snapshot.scratch(B)
        nat.call("mpv_snapshot_forward", ctypes_byref(self.snapshot.struct), packed.data_ptr(), B,
                 out.data_ptr(), None, None, status.data_ptr(), scratch.data_ptr(), scratch.numel(),
                 nat.stream_handle(self.device))
        return out, status

    def __call__(self, bits) -> np.ndarray:
        import torch

        bits = np.atleast_2d(np.asarray(bits, dtype=np.uint8))
        if bits.shape[1] != self.n_visible:
            raise ValueError(f"bit matrix has {bits.shape[1]} sites, ansatz has {self.n_visible}")
        packed = device_pack(bits, self.device)
        out, status = self.log_prob_packed(packed)
        out = out.cpu().numpy()
        _raise_nonfinite(status, bits, "log probability")
        return out


class LogPsiEvaluator:
    """f64 log-amplitude evaluator ``uint8[B,N] -> complex128[B]`` with the
    master parameters (rbm.py:419-425); also carries the parameters the
    device local-energy kernel needs."""

    def __init__(self, params: RbmParameters, device=None):
        self.params = params
        self.snapshot = DeviceSnapshot(params, F64, RoundingMode.PER_OPERATION, device)
        self.device = self.snapshot.device
        self._energy_cache = {}

    def log_psi_packed(self, packed):
        import torch

        B = packed.shape[0]
        lp = torch.empty(B, dtype=torch.float64, device=self.device)
        re = torch.empty_like(lp)
        im = torch.empty_like(lp)
        status = _status_tensor(self.device)
        nat.call("mpv_snapshot_forward", ctypes_byref(self.snapshot.struct), packed.data_ptr(), B,
                 lp.data_ptr(), re.data_ptr(), im.data_ptr(), status.data_ptr(), None, 0,
                 nat.stream_handle(self.device))
        return re, im, status

    def __call__(self, bits) -> np.ndarray:
        import torch

        bits = np.atleast_2d(np.asarray(bits, dtype=np.uint8))
        if bits.shape[1] != self.snapshot.n_visible:
            raise ValueError(f"bit matrix has {bits.shape[1]} sites, ansatz has {self.snapshot.n_visible}")
        packed = device_pack(bits, self.device)
        re, im, status = self.log_psi_packed(packed)
        out = re.cpu().numpy() + 1j * im.cpu().numpy()
        _raise_nonfinite(status, bits, "log psi")
        return out


def ctypes_byref(struct):
    import ctypes

    return ctypes.byref(struct)


def _raise_nonfinite(status, bits, what):
    st = status.cpu().numpy()
    if st[0] != 0:
        bad = int(st[1])
        raise EvaluationFailureError(f"non-finite {what} for configuration bits {bits[bad].tolist()}",
                                     context={"bits": bits[bad].copy()})


@dataclass(frozen=True)
class NoiseField:
    """Frozen Gaussian log-density noise: std sigma, fixed per (seed, x)
    (rbm.py:333-352).  On the device it is added inside the f64 sweep and the
    forward (mpv_snapshot noise_key / noise_sigma)."""

    sigma: float
    seed: int

    def __post_init__(self):
        if self.sigma < 0:
            raise ValueError("sigma must be >= 0")

    @property
    def key(self):
        return derive_key(self.seed, "noise-field")

    def zeta(self, codes) -> np.ndarray:
        """delta(x) = zeta(x) for configuration codes (host; rbm.py:347-352)."""
        codes = np.asarray(codes, dtype=np.uint64)
        if self.sigma == 0.0:
            return np.zeros(codes.shape)
        return gaussian_field(self.key, codes, self.sigma)


def noisy_log_prob_evaluator(params, noise: NoiseField, device=None) -> LogProbEvaluator:
    """f64 log-probability plus the frozen noise field (rbm.py:408-416), as a
    device evaluator: ChainEnsemble runs the fused f64 sweep with the noise
    added to every proposal's log p (N <= 64, like the reference's codes)."""
    if params.n_visible > 64:
        raise ValueError("noise fields are keyed by 64-bit configuration codes (n_visible <= 64)")
    ev = LogProbEvaluator(params, F64, RoundingMode.PER_OPERATION, device)
    ev.noise = noise
    ev.snapshot.struct.noise_key = int(noise.key)
    ev.snapshot.struct.noise_sigma = float(noise.sigma)
    return ev


def log_prob_evaluator(params, fmt: FloatFormat = F64, mode: RoundingMode = RoundingMode.PER_OPERATION,
                       device=None, variant: int | None = None) -> LogProbEvaluator:
    """Device log-probability evaluator (rbm.py:361-405); parameters are
    downcast once at construction.  ``mode=RoundingMode.NATIVE`` selects the
    B200 fused-sweep arithmetic; ``variant`` overrides the
    exact-accumulator planner (all valid variants give identical results)."""
    return LogProbEvaluator(params, fmt, mode, device, variant)


def log_psi_evaluator(params, device=None) -> LogPsiEvaluator:
    return LogPsiEvaluator(params, device)


def log_prob_batch(params, bits, fmt: FloatFormat = F64, mode: RoundingMode = RoundingMode.PER_OPERATION,
                   device=None) -> np.ndarray:
    """log p(x) for a (B, N) bit matrix (rbm.py:276-296)."""
    bits = np.atleast_2d(np.asarray(bits))
    if bits.shape[1] != params.n_visible:
        raise ValueError(f"bit matrix has {bits.shape[1]} sites, ansatz has {params.n_visible}")
    return LogProbEvaluator(params, fmt, mode, device)(bits)


def log_psi_batch(params, bits, fmt: FloatFormat = F64, mode: RoundingMode = RoundingMode.PER_OPERATION,
                  device=None) -> np.ndarray:
    """log psi(x) (rbm.py:254-273): f64 / storage-only via the f64 kernel on
    the (rounded) parameters, per-operation via the emulation kernel."""
    import torch

    bits = np.atleast_2d(np.asarray(bits, dtype=np.uint8))
    if bits.shape[1] != params.n_visible:
        raise ValueError(f"bit matrix has {bits.shape[1]} sites, ansatz has {params.n_visible}")
    if fmt.name == "f64" or mode is RoundingMode.STORAGE_ONLY:
        return LogPsiEvaluator(round_parameters(params, fmt), device)(bits)
    if mode is RoundingMode.NATIVE:
        raise ValueError("NATIVE mode computes log p only (use log_prob_batch)")
    snap = DeviceSnapshot(params, fmt, mode, device)
    packed = device_pack(bits, snap.device)
    B = bits.shape[0]
    lp = torch.empty(B, dtype=torch.float64, device=snap.device)
    re, im = torch.empty_like(lp), torch.empty_like(lp)
    status = _status_tensor(snap.device)
    nat.call("mpv_snapshot_forward", ctypes_byref(snap.struct), packed.data_ptr(), B, lp.data_ptr(),
             re.data_ptr(), im.data_ptr(), status.data_ptr(), None, 0, nat.stream_handle(snap.device))
    out = re.cpu().numpy() + 1j * im.cpu().numpy()
    _raise_nonfinite(status, bits, "log psi")
    return out


class TensorCoreForward:
    """Batched forward of the RBM as a tcgen05 tensor-core GEMM (north_star
    subsystem (2)): theta = b + W x with f16/bf16 operands (the parameters
    rounded as round_parameters, rbm.py:91-101; x in {0,1} exact) and f32
    accumulators in TMEM, the log-cosh sum of rbm.py:130-150 as the GEMM's
    epilogue.  Agrees with the f64 forward of the rounded parameters to f32
    accumulation error; the sampler's bit-exact arithmetics (per-operation,
    NATIVE) stay in the sweep kernels."""

    def __init__(self, params: RbmParameters, fmt: FloatFormat, device=None):
        import torch

        nat.require_cuda()
        if fmt.name not in ("f16", "bf16"):
            raise ValueError("the tensor-core forward takes f16 or bf16 parameters")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.params, self.fmt = params, fmt
        N, M = params.n_visible, params.n_hidden
        self.n_visible, self.n_hidden = N, M
        nbytes = int(nat.load().mpv_forward_tc_weights_bytes(N, M))
        if nbytes == 0:
            raise ValueError(f"tensor-core forward: unsupported shape N={N}, M={M}")
        host = torch.empty(2 * (N + M + N * M), dtype=torch.float64, pin_memory=True)
        hv = host.numpy().view(np.complex128)
        hv[:N], hv[N:N + M] = params.a, params.b
        hv[N + M:].reshape(N, M)[:] = params.w.T
        src = host.to(self.device, non_blocking=True)
        self._weights = torch.zeros(nbytes, dtype=torch.uint8, device=self.device)
        nat.call("mpv_forward_tc_prepare", N, M, fmt.code, src.data_ptr(), self._weights.data_ptr(),
                 nat.stream_handle(self.device))
        torch.cuda.current_stream(self.device).synchronize()  # `host`/`src` are released on return

    def forward_packed(self, packed, out_lp=None, out_re=None, out_im=None, max_ctas: int = 0):
        """Device call on packed words [B, ceil(N/32)]; returns (lp, re, im) f64 tensors."""
        import torch

        words = (self.n_visible + 31) // 32
        if packed.dtype not in (torch.int32, torch.uint32) or packed.dim() != 2 or packed.shape[1] != words:
            raise ValueError(f"packed configurations must be an int32 [B, {words}] tensor, got "
                             f"{packed.dtype} {tuple(packed.shape)}")
        if not packed.is_contiguous() or packed.device != self.device:
            raise ValueError("packed configurations must be contiguous and on the evaluator's device")
        B = packed.shape[0]
        for t in (out_lp, out_re, out_im):
            if t is not None and (t.dtype != torch.float64 or t.numel() < B or not t.is_contiguous()
                                  or t.device != self.device):
                raise ValueError("outputs must be contiguous float64 device tensors with >= B elements")
        if out_lp is None and out_re is None and out_im is None:
            out_lp = torch.empty(B, dtype=torch.float64, device=self.device)
            out_re, out_im = torch.empty_like(out_lp), torch.empty_like(out_lp)
        ptr = (lambda t: t.data_ptr() if t is not None else None)
        nat.call("mpv_forward_tc", self.n_visible, self.n_hidden, self.fmt.code, self._weights.data_ptr(),
                 packed.data_ptr(), B, ptr(out_lp), ptr(out_re), ptr(out_im), int(max_ctas),
                 nat.stream_handle(self.device))
        return out_lp, out_re, out_im

    def __call__(self, bits) -> np.ndarray:
        """complex128 log psi for a (B, N) uint8 bit matrix."""
        bits = np.atleast_2d(np.asarray(bits, dtype=np.uint8))
        if bits.shape[1] != self.n_visible:
            raise ValueError(f"bit matrix has {bits.shape[1]} sites, ansatz has {self.n_visible}")
        _, re, im = self.forward_packed(device_pack(bits, self.device))
        return re.cpu().numpy() + 1j * im.cpu().numpy()


def log_psi_batch_tc(params, bits, fmt: FloatFormat, device=None) -> np.ndarray:
    """log psi(x) for a (B, N) bit matrix through the tensor-core forward."""
    return TensorCoreForward(params, fmt, device)(bits)


# ---------------------------------------------------------------------------
# delta-distribution studies (rbm.py:429-492): delta(x) = log p_fmt - log p_f64
# evaluated on the device over the full enumeration; summaries on the host.
# ---------------------------------------------------------------------------

@dataclass(frozen=True)
class DeltaSummary:
    """Moments of delta over the enumerated space plus its Shapiro-Wilk W."""

    mean: float
    std: float
    skewness: float
    excess_kurtosis: float
    shapiro_wilk_w: float
    shapiro_n: int


def precision_delta(params, fmt, mode, bits) -> np.ndarray:
    """delta on an arbitrary batch (rbm.py:472-474), both evaluations on the device."""
    return log_prob_batch(params, bits, fmt, mode) - log_prob_batch(params, bits, F64)


def delta_distribution(params, fmt, mode, lattice_spec):
    """(DeltaSummary, delta vector) over the full enumeration (rbm.py:440-469);
    Shapiro-Wilk on the standardised field, deterministically subsampled to
    5000 points by the reference's counter-based order."""
    from .lattice import enumerate_bits
    from .normality import shapiro_wilk, standardize
    from .rng import counter_uniform

    bits = enumerate_bits(lattice_spec.n_sites)
    delta = precision_delta(params, fmt, mode, bits)
    mean, std = float(delta.mean()), float(delta.std())
    if std == 0.0:
        return DeltaSummary(mean, 0.0, 0.0, 0.0, float("nan"), 0), delta
    z = standardize(delta)
    sample = z
    if sample.size > 5000:
        order = np.argsort(counter_uniform(derive_key(0, "sw-subsample"), np.arange(sample.size)))
        sample = sample[order[:5000]]
    report = shapiro_wilk(sample)
    return DeltaSummary(mean, std, float((z**3).mean()), float((z**4).mean() - 3.0), report.w, report.n), delta


def delta_for_noise(params, noise: NoiseField, n: int) -> np.ndarray:
    """delta induced by a frozen noise field over the full enumeration (rbm.py:477-480)."""
    return noise.zeta(np.arange(1 << n, dtype=np.uint64))
