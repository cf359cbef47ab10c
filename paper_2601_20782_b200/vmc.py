"""Local energies and the per-iteration estimators on the B200 (mirror of the
reference vmc.py:52-131, 311-317).

``local_energies(spec, log_amplitude, bits)`` keeps the reference signature;
``log_amplitude`` must be a device evaluator from ``rbm.log_psi_evaluator``
(it carries the f64 master parameters the kernel needs).  The kernel
(csrc/energy.cuh) evaluates every connected amplitude ratio as an O(M)
product instead of a full forward pass per connected configuration.
"""
from __future__ import annotations

import ctypes

import numpy as np

from . import _native as nat
from .errors import DegenerateInputError, EvaluationFailureError
from .hamiltonians import HeisenbergSpec, J1J2Spec, TfimSpec
from .lattice import pack_bits


class EnergyKernel:
    """Device parameters + cosh/sinh tables of one (params, Hamiltonian) pair."""

    def __init__(self, spec, params, device=None):
        import torch

        nat.require_cuda()
        coef = bond_j = None
        if isinstance(spec, TfimSpec):
            self.ham, self.J, self.h = nat.HAM_TFIM, float(spec.j), float(spec.h)
            bonds = spec.lattice.bond_array()
        elif isinstance(spec, (HeisenbergSpec, J1J2Spec)):
            self.ham, self.h = nat.HAM_HEISENBERG, 0.0
            self.J = float(spec.j) if isinstance(spec, HeisenbergSpec) else float(spec.j1)
            bonds, jb, cf = spec.couplings()
            if isinstance(spec, J1J2Spec) or spec.marshall:  # general couplings (mpv_local_energies_ex)
                coef, bond_j = cf, jb
        else:
            raise TypeError(f"unknown Hamiltonian spec {type(spec).__name__}")
        n = spec.lattice.n_sites
        if params.n_visible != n:
            raise ValueError(f"ansatz has {params.n_visible} sites, lattice has {n}")
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.N, self.M = n, params.n_hidden
        cplx = lambda z: torch.from_numpy(np.ascontiguousarray(np.stack([z.real, z.imag], -1))).to(self.device)
        self.a = cplx(params.a)
        self.b = cplx(params.b)
        self.w_t = cplx(np.ascontiguousarray(params.w.T))
        bonds = bonds.astype(np.int32)
        self.n_bonds = bonds.shape[0]
        f64 = lambda v: torch.from_numpy(np.ascontiguousarray(v, dtype=np.float64)).to(self.device)
        self.term_coef = f64(coef) if coef is not None else None
        self.bond_j = f64(bond_j) if bond_j is not None else None
        self.bonds = torch.from_numpy(np.ascontiguousarray(bonds.reshape(-1))).to(self.device) if self.n_bonds else None
        nbytes = nat.load().mpv_energy_tables_bytes(self.N, self.M, self.ham, self.n_bonds)
        self.tables = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        nat.call("mpv_energy_prepare", self.N, self.M, self.a.data_ptr(), self.b.data_ptr(), self.w_t.data_ptr(),
                 self.ham, self._bonds_ptr(), self.n_bonds, self.tables.data_ptr(), nat.stream_handle(self.device))

    def _bonds_ptr(self):
        return self.bonds.data_ptr() if self.bonds is not None else None

    def packed(self, packed_bits):
        """Device path: packed configurations -> (complex128-as-(B,2) f64 tensor, status tensor)."""
        import torch

        B = packed_bits.shape[0]
        out = torch.empty((B, 2), dtype=torch.float64, device=self.device)
        status = torch.tensor([0, 2**63 - 1], dtype=torch.int64, device=self.device)
        ptr = lambda t: t.data_ptr() if t is not None else None
        nat.call("mpv_local_energies_ex", self.N, self.M, self.a.data_ptr(), self.b.data_ptr(), self.w_t.data_ptr(),
                 self.ham, self._bonds_ptr(), self.n_bonds, self.J, self.h, ptr(self.term_coef), ptr(self.bond_j),
                 self.tables.data_ptr(), packed_bits.data_ptr(), B, out.data_ptr(), status.data_ptr(),
                 nat.stream_handle(self.device))
        return out, status


def _energy_kernel(spec, log_amplitude):
    from .rbm import LogPsiEvaluator

    if not isinstance(log_amplitude, LogPsiEvaluator):
        raise TypeError("local_energies needs a device evaluator from rbm.log_psi_evaluator "
                        f"(got {type(log_amplitude).__name__}; there is no host-callable fallback)")
    key = spec  # frozen dataclasses: hashable, equal specs share the tables
    cache = log_amplitude._energy_cache
    if key not in cache:
        cache[key] = EnergyKernel(spec, log_amplitude.params, log_amplitude.device)
    return cache[key]


def local_energies(spec, log_amplitude, bits) -> np.ndarray:
    """eps(x) = sum_{x'} H(x, x') psi(x')/psi(x) for a (S, N) bit matrix (vmc.py:60-108)."""
    import torch

    kern = _energy_kernel(spec, log_amplitude)
    bits = np.atleast_2d(np.asarray(bits, dtype=np.uint8))
    if bits.shape[1] != kern.N:
        raise ValueError(f"bit matrix has {bits.shape[1]} sites, lattice has {kern.N}")
    from .rbm import device_pack

    packed = device_pack(bits, kern.device)
    out, status = kern.packed(packed)
    host = torch.empty((out.shape[0] + 1, 2), dtype=torch.float64, pin_memory=True)
    host[:-1].copy_(out, non_blocking=True)
    host[-1:].view(torch.int64).copy_(status.view(1, 2), non_blocking=True)
    torch.cuda.current_stream(kern.device).synchronize()
    eps = host[:-1].numpy()
    st = host[-1:].view(torch.int64).numpy()[0]
    if st[0] != 0:
        bad = int(st[1])
        raise EvaluationFailureError("non-finite local energy", context={"bits": bits[bad].copy()})
    return eps[:, 0] + 1j * eps[:, 1]


def local_energy(spec, log_amplitude, x) -> complex:
    bits = x.bits()[None, :] if hasattr(x, "bits") and callable(x.bits) else np.atleast_2d(x)
    return complex(local_energies(spec, log_amplitude, bits)[0])


def mc_error(values) -> float:
    """sqrt(sample variance / N) with the unbiased variance (vmc.py:311-317)."""
    values = np.asarray(values, dtype=np.float64)
    if values.size < 2:
        raise DegenerateInputError("need >= 2 values")
    return float(np.sqrt(values.var(ddof=1) / values.size))


# ---------------------------------------------------------------------------
# Training loop: two-copy mixed-precision SR (mirror of the reference
# vmc.py:145-229, 320-639).  Sampling and local energies run in the CUDA
# library; the f64 statistics O, F, S and the SR solve stay in f64 on the
# device (torch / cuBLAS / cuSOLVER library calls: plain GEMM/Cholesky).
# ---------------------------------------------------------------------------
import time  # noqa: E402
from dataclasses import dataclass, field  # noqa: E402
from fractions import Fraction  # noqa: E402

from .errors import SolverError  # noqa: E402
from .precision import F64, FloatFormat, RoundingMode  # noqa: E402


def _t(x, device):
    import torch

    return torch.as_tensor(np.asarray(x), device=device)


def grad_log_psi_device(params, bits_u8, device=None):
    """O(x) = d log psi / d theta (rbm.py:307-325) for a (U, N) uint8 device
    tensor: columns a, b, W row-major; complex128 [U, P] on the device."""
    import torch

    dev = bits_u8.device
    x = bits_u8.to(torch.float64).to(torch.complex128)
    w = _t(params.w, dev)
    b = _t(params.b, dev)
    th = x @ w.T + b[None, :]
    t = torch.tanh(th)
    U, N = x.shape
    M = b.numel()
    out = torch.empty((U, N + M + M * N), dtype=torch.complex128, device=dev)
    out[:, :N] = x
    out[:, N:N + M] = t
    out[:, N + M:] = (t[:, :, None] * x[:, None, :]).reshape(U, M * N)
    return out


def forces(*, o, eps, weights=None):
    """F_k = E[conj(O_k) eps] - E[conj(O_k)] E[eps] (vmc.py:145-165), device tensors."""
    if o.shape[0] != eps.numel() or eps.numel() == 0:
        raise DegenerateInputError("need at least one (O, eps) pair")
    oc = o.conj()
    if weights is None:
        if eps.numel() < 2:
            raise DegenerateInputError("need >= 2 samples")
        return oc.T @ eps / eps.numel() - oc.mean(dim=0) * eps.mean()
    w = weights.to(oc.dtype)
    return (oc * w[:, None]).T @ eps - (w @ oc) * (w @ eps)


def s_matrix(*, o, weights=None):
    """S = E[conj(O) O^T] - E[conj O] E[O^T], Hermitised (vmc.py:168-188)."""
    if o.shape[0] == 0:
        raise DegenerateInputError("empty sample set")
    if weights is None:
        c = o - o.mean(dim=0, keepdim=True)
        s = c.conj().T @ c / o.shape[0]
    else:
        w = weights.to(o.dtype)
        mean = w @ o
        c = o - mean[None, :]
        s = c.conj().T @ (c * w[:, None])
    return 0.5 * (s + s.conj().T)


@dataclass(frozen=True)
class SrUpdate:
    g: object
    kappa: float
    residual: float
    lambda_shift: float
    eta: float
    iterations: int = 0  # conjugate-gradient iterations (matrix-free solver)


def sr_step(f, s, lambda_shift: float, eta: float, compute_kappa: bool = True) -> SrUpdate:
    """(S + lambda I) g = F by Cholesky + one refinement pass (vmc.py:202-229)."""
    import torch

    if lambda_shift < 0:
        raise ValueError("lambda must be >= 0")
    if eta <= 0:
        raise ValueError("eta must be > 0")
    shifted = s + lambda_shift * torch.eye(s.shape[0], dtype=s.dtype, device=s.device)
    L, info = torch.linalg.cholesky_ex(shifted)
    if int(info) != 0:
        smallest = float(torch.linalg.eigvalsh(shifted)[0])
        raise SolverError(f"shifted S is not positive definite (smallest eigenvalue {smallest:.3e})")
    g = torch.cholesky_solve(f[:, None], L)[:, 0]
    g = g + torch.cholesky_solve((f - shifted @ g)[:, None], L)[:, 0]
    kappa = float("nan")
    if compute_kappa:
        ev = torch.linalg.eigvalsh(shifted)
        kappa = float(ev[-1] / ev[0]) if float(ev[0]) > 0 else float("inf")
    fn = float(torch.linalg.norm(f))
    residual = float(torch.linalg.norm(shifted @ g - f)) / fn if fn > 0 else 0.0
    if fn > 0 and residual > 1e-10:
        raise SolverError(f"SR solve residual {residual:.3e} exceeds 1e-10")
    return SrUpdate(g, kappa, residual, lambda_shift, eta)


class FactoredLogDerivatives:
    """O(x) = [x, tanh(theta), tanh(theta) (x) x] (rbm.py:307-325) kept in factored
    form: the packed sample bits X and T = tanh(b + W x) (U, M) complex, never
    the (U, P) matrix (P = N + M + M N is 20,300 at config 2: O would be 21 GB
    and S 6.6 GB).  O v and O^H u run in csrc/logderiv.cuh as DMMA GEMMs over
    the bits with fused epilogues (mpv_logderiv_ov / mpv_logderiv_ohu).
    `reduce` (optional) all-reduces sums over samples across ranks."""

    def __init__(self, params, bits_u8, packed=None, reduce=None):
        import torch

        dev = bits_u8.device
        self.N, self.M = params.n_visible, params.n_hidden
        self.U = bits_u8.shape[0]
        if packed is None:
            packed = torch.empty((self.U, (self.N + 31) // 32), dtype=torch.int32, device=dev)
            if self.U:
                nat.call("mpv_pack_bits", bits_u8.data_ptr(), self.U, self.N, packed.data_ptr(), nat.stream_handle(dev))
        self.packed = packed.contiguous()
        self.packed_u8 = bits_u8
        x = bits_u8.to(torch.complex128)
        self.t = torch.tanh(x @ _t(params.w, dev).T + _t(params.b, dev)[None, :]).contiguous()
        self.scratch = torch.empty(nat.load().mpv_logderiv_scratch_bytes(self.U, self.N, self.M), dtype=torch.uint8,
                                   device=dev)
        self.reduce = reduce or (lambda z: z)
        self.reduce_is_local = reduce is None
        self.device = dev

    def o_v(self, v):
        import torch

        v = v.contiguous()
        q = torch.empty(self.U, dtype=torch.complex128, device=self.device)
        nat.call("mpv_logderiv_ov", self.t.data_ptr(), self.packed.data_ptr(), self.U, self.N, self.M, v.data_ptr(),
                 q.data_ptr(), self.scratch.data_ptr(), nat.stream_handle(self.device))
        return q

    def oh_u(self, u):
        """sum_s conj(O_s) u_s (local sums; callers reduce)."""
        import torch

        u = u.contiguous()
        out = torch.empty(self.N + self.M + self.M * self.N, dtype=torch.complex128, device=self.device)
        nat.call("mpv_logderiv_ohu", self.t.data_ptr(), self.packed.data_ptr(), self.U, self.N, self.M, u.data_ptr(),
                 out.data_ptr(), self.scratch.data_ptr(), nat.stream_handle(self.device))
        return out


def sr_step_cg(o: FactoredLogDerivatives, eps, weights, lambda_shift: float, eta: float,
               tol: float = 1e-10, maxiter: int = 1000):
    """SR update without forming S (matrix-free conjugate gradients on the
    Hermitian positive-definite S + lambda I; beyond the
    reference's dense Cholesky, vmc.py:202-229, which does not fit config 2).
    Same estimators: F = sum_w conj(O) eps - (sum_w conj O)(sum_w eps),
    S v = sum_w conj(O) (O v) - conj(Obar)(Obar v).  Returns (SrUpdate, F, energy)."""
    import torch

    if lambda_shift < 0:
        raise ValueError("lambda must be >= 0")
    if eta <= 0:
        raise ValueError("eta must be > 0")
    w = weights.to(torch.complex128)
    s_oe = o.reduce(o.oh_u(w * eps))
    s_o = o.reduce(o.oh_u(w))
    e = o.reduce((w @ eps).reshape(1))[0]
    f = s_oe - s_o * e
    obar = s_o.conj()  # sum_w O

    def apply(v):
        return o.reduce(o.oh_u(w * o.o_v(v))) - obar.conj() * (obar @ v) + lambda_shift * v

    g = torch.zeros_like(f)
    r = f.clone()
    pvec = r.clone()
    rr = torch.vdot(r, r).real
    fn = float(torch.linalg.norm(f))
    it = 0
    while it < maxiter and fn > 0 and float(rr) ** 0.5 > tol * fn:
        ap = apply(pvec)
        alpha = rr / torch.vdot(pvec, ap).real
        g = g + alpha * pvec
        r = r - alpha * ap
        rr_new = torch.vdot(r, r).real
        pvec = r + (rr_new / rr) * pvec
        rr = rr_new
        it += 1
    residual = float(torch.linalg.norm(apply(g) - f)) / fn if fn > 0 else 0.0
    if fn > 0 and residual > max(10 * tol, 1e-9):
        raise SolverError(f"SR conjugate-gradient residual {residual:.3e} after {it} iterations")
    return SrUpdate(g, float("nan"), residual, lambda_shift, eta, it), f, float(e.real)


def sr_step_minsr(o: FactoredLogDerivatives, eps, weights, lambda_shift: float, eta: float):
    """The same SR update solved in sample space (minSR; beyond the reference).

    With O~ = W^{1/2} (O - 1 obar^T) the reference's estimators are S = O~^H O~
    and F = O~^H e~ (e~ = W^{1/2} (eps - ebar)), and the push-through identity
    gives g = (S + lambda)^-1 F = O~^H (O~ O~^H + lambda)^-1 e~ exactly: a U x U
    Cholesky instead of a P x P one (cheaper whenever U < P).  The Gram matrix
    never needs O: O O^H = X X^T + (T T^H) * (1 + X X^T) (elementwise), one real
    and one complex GEMM (cuBLAS); O^H y runs in csrc/logderiv.cuh.
    Single process only (the U x U system couples every rank's samples)."""
    import torch

    if lambda_shift < 0:
        raise ValueError("lambda must be >= 0")
    if eta <= 0:
        raise ValueError("eta must be > 0")
    if not o.reduce_is_local:
        raise ValueError("minSR couples all samples: use sr_solver='cg' or 'dense' across ranks")
    w = weights.to(torch.float64)
    wc = w.to(torch.complex128)
    obar = o.oh_u(wc).conj()  # sum_w O
    e = wc @ eps
    xr = o.packed_u8.to(torch.float64)
    xx = xr @ xr.T
    gram = xx.to(torch.complex128) + (o.t @ o.t.mH) * (1.0 + xx)
    c = o.o_v(obar.conj())  # c_s = sum_j O_sj conj(obar_j)
    ones = torch.ones_like(c)
    k = gram - c[:, None] * ones[None, :] - ones[:, None] * c.conj()[None, :] + torch.vdot(obar, obar).real
    sw = torch.sqrt(w).to(torch.complex128)
    k = sw[:, None] * k * sw[None, :]
    k = 0.5 * (k + k.mH)
    k += lambda_shift * torch.eye(k.shape[0], dtype=k.dtype, device=k.device)
    et = sw * (eps - e)
    L, info = torch.linalg.cholesky_ex(k)
    if int(info) != 0:
        raise SolverError("sample-space matrix O~ O~^H + lambda I is not positive definite")
    y = torch.cholesky_solve(et[:, None], L)[:, 0]
    y = y + torch.cholesky_solve((et - k @ y)[:, None], L)[:, 0]  # one refinement pass
    z = sw * y
    g = o.oh_u(z) - obar.conj() * z.sum()
    f = o.oh_u(wc * eps) - o.oh_u(wc) * e
    residual = float(torch.linalg.norm(k @ y - et) / max(float(torch.linalg.norm(et)), 1e-300))
    return SrUpdate(g, float("nan"), residual, lambda_shift, eta), f, float(e.real)


@dataclass
class TrainConfig:
    """Reference TrainConfig (vmc.py:320-351) plus compute_kappa (the eigvalsh of
    S + lambda I is O(P^3); large-P runs may switch it off)."""

    hamiltonian: object
    alpha: object = 1
    n_steps: int = 500
    n_samples: int = 4096
    eta: float = 0.01
    lambda_shift: float = 1e-3
    seed: int = 0
    sampling_format: FloatFormat = F64
    rounding_mode: RoundingMode = RoundingMode.PER_OPERATION
    sampling_mode: str = "mcmc"
    proposal: object = None
    n_chains: int | None = None
    burn_in_sweeps: int | None = None
    reburn_sweeps: int = 2
    thin_sweeps: int = 1
    log_every: int = 1
    init_scale: float = 0.01
    track_forces: bool = False
    track_timings: bool = False
    reference_energy: float | None = None
    compute_kappa: bool = True
    sr_solver: str = "dense"  # "dense" (reference: Cholesky on S), "cg" (matrix-free) or "minsr" (sample space)
    cg_tol: float = 1e-10
    cg_maxiter: int = 1000

    def __post_init__(self):
        if self.n_steps < 1 or self.n_samples < 2:
            raise ValueError("n_steps and n_samples must be positive")
        if self.sampling_mode not in ("mcmc", "exact"):
            raise ValueError(f"unknown sampling mode {self.sampling_mode!r}")
        if self.sr_solver not in ("dense", "cg", "minsr"):
            raise ValueError(f"unknown SR solver {self.sr_solver!r}")
        if self.proposal is None:
            from .sampler import Proposal

            self.proposal = Proposal("flip")


@dataclass
class TrainResult:
    records: list
    params: object
    force_history: list = field(default_factory=list)


def train(config: TrainConfig, device=None, group=None, local: bool = False) -> TrainResult:
    """Two-copy mixed-precision SR training (vmc.py:472-639) on the device.

    Under torch.distributed (world > 1) each rank samples its contiguous slice
    of the global chains (draws depend on global chain ids only), evaluates
    local energies and O on its own samples, and the forces, S-matrix, energy,
    split-chain error and acceptance come from all-reduces
    (parallel.sharded_statistics / energy_statistics); every rank then solves
    the same SR system.  sigma-hat pools per-rank deduplicated batches."""
    import torch
    import torch.distributed as tdist

    from . import parallel

    from . import rbm
    from .bounds import pinsker_tv_bound, theorem3_gaussian_bound
    from .lattice import enumerate_bits, unpack_bits
    from .rng import derive_key
    from .sampler import ChainEnsemble, default_chain_count

    nat.require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    # local=True: a single-process run even inside an initialised process group
    world = tdist.get_world_size(group) if (not local and tdist.is_available() and tdist.is_initialized()) else 1
    exact_mode = config.sampling_mode == "exact"
    if exact_mode:
        # every rank enumerates the whole space with globally normalised weights;
        # summing those across ranks would count each configuration `world` times,
        # so exact mode runs the (identical) single-process update on every rank
        world = 1
    rank = tdist.get_rank(group) if world > 1 else 0
    spec = config.hamiltonian
    n = spec.lattice.n_sites
    params = rbm.random_parameters(n, Fraction(config.alpha), derive_key(config.seed, "init"), config.init_scale)
    n_chains = config.n_chains or default_chain_count(config.n_samples)
    burn_in = config.burn_in_sweeps if config.burn_in_sweeps is not None else 10 * n
    words = (n + 31) // 32
    if exact_mode:
        from .lattice import pack_bits

        all_u8 = enumerate_bits(n)
        all_packed = torch.from_numpy(pack_bits(all_u8)).to(dev)
    else:
        c_off, c_cnt = parallel.shard(n_chains, rank, world)
        counts = parallel.chain_counts(config.n_samples, n_chains, c_off, c_cnt)
        chain_ids = torch.as_tensor(np.repeat(np.arange(c_cnt), counts), device=dev)
        per_chain = torch.as_tensor(counts, device=dev, dtype=torch.float64)
    ensemble = None
    records, force_history = [], []
    for step in range(config.n_steps):
        torch.cuda.synchronize(dev)
        t_sample = time.perf_counter()
        nvtx = torch.cuda.nvtx  # phase ranges for nsys/ncu timelines (no-ops without a profiler)
        nvtx.range_push(f"vmc step {step}: sampling")
        if exact_mode:
            lp = rbm.LogProbEvaluator(params, F64, RoundingMode.PER_OPERATION, dev).log_prob_packed(all_packed)[0]
            weights = torch.softmax(lp, dim=0)
            uniq = all_packed
            est_w = weights
            acceptance = float("nan")
            ev = None
        else:
            ev = rbm.log_prob_evaluator(params, config.sampling_format, config.rounding_mode, dev)
            if ensemble is None:
                ensemble = ChainEnsemble(c_cnt, n, config.proposal, ev, derive_key(config.seed, "chains"),
                                         chain_offset=c_off, n_chains_total=n_chains)
                ensemble.run_sweeps(burn_in)
            else:
                ensemble.set_evaluator(ev)
                ensemble.run_sweeps(config.reburn_sweeps)
            ensemble.reset_counters()
            packed = ensemble.collect_packed(config.n_samples, config.thin_sweeps * n + 1)
            acceptance = ensemble.acceptance_rate
            if world > 1:
                ap = torch.tensor([float(ensemble.accepted), float(ensemble.proposed)], dtype=torch.float64,
                                  device=dev)
                parallel.all_reduce_sum(ap, group)
                acceptance = float(ap[0] / ap[1])
            # np.unique(..., axis=0) over the sample stream (vmc.py:560-563)
            uniq, inverse, cnt = torch.unique(packed, dim=0, return_inverse=True, return_counts=True)
            est_w = cnt.to(torch.float64) / config.n_samples
        torch.cuda.synchronize(dev)
        t_update = time.perf_counter()
        nvtx.range_pop()
        nvtx.range_push(f"vmc step {step}: energies + SR update")
        psi = rbm.log_psi_evaluator(params, dev)
        eps_ri, status = _energy_kernel(spec, psi).packed(uniq)
        if int(status[0]) != 0:
            raise EvaluationFailureError("non-finite local energy", context={"step": step})
        eps = torch.complex(eps_ri[:, 0], eps_ri[:, 1])
        u8 = torch.empty((uniq.shape[0], n), dtype=torch.uint8, device=dev)
        nat.call("mpv_unpack_bits", uniq.data_ptr(), uniq.shape[0], n, u8.data_ptr(), nat.stream_handle(dev))
        if config.sr_solver == "cg":
            red = (lambda z: parallel.all_reduce_sum(z, group)) if world > 1 else None
            fo = FactoredLogDerivatives(params, u8, uniq, red)
            update, f, energy = sr_step_cg(fo, eps, est_w, config.lambda_shift, config.eta, config.cg_tol,
                                           config.cg_maxiter)
        elif config.sr_solver == "minsr":
            if world > 1:
                raise ValueError("sr_solver='minsr' is single-process (use 'cg' or 'dense' across ranks)")
            update, f, energy = sr_step_minsr(FactoredLogDerivatives(params, u8, uniq), eps, est_w,
                                              config.lambda_shift, config.eta)
        else:
            o = grad_log_psi_device(params, u8)
            if world > 1:
                f, s, e_glob = parallel.sharded_statistics(o, eps, est_w, group)
                energy = float(e_glob)
            else:
                f = forces(o=o, eps=eps, weights=est_w)
                s = s_matrix(o=o, weights=est_w)
                energy = float((est_w.to(eps.dtype) @ eps).real)
            update = sr_step(f, s, config.lambda_shift, config.eta, config.compute_kappa)
        theta = params.flatten() - config.eta * update.g.cpu().numpy()
        nvtx.range_pop()
        new_params = rbm.RbmParameters.from_flat(theta, params.n_visible, params.n_hidden)
        if exact_mode:
            err = 0.0
        elif world > 1:
            err = parallel.energy_statistics(eps.real[inverse], counts, 0, 1, group)["mc_error"]
        else:
            stream = eps.real[inverse]
            if n_chains > 1:
                sums = torch.zeros(n_chains, dtype=torch.float64, device=dev).index_add_(0, chain_ids, stream)
                err = mc_error((sums / per_chain).cpu().numpy())
            else:
                err = mc_error(stream.cpu().numpy())
        if config.track_forces:
            force_history.append(f.cpu().numpy())
        if step % config.log_every == 0 or step == config.n_steps - 1:
            if exact_mode or config.sampling_format.name == "f64":
                sigma_hat = 0.0
            else:
                lp_fmt, _ = ev.log_prob_packed(uniq)
                lp64 = rbm.LogProbEvaluator(params, F64, RoundingMode.PER_OPERATION, dev).log_prob_packed(uniq)[0]
                delta = lp_fmt - lp64
                if world > 1:
                    mom = torch.stack([delta.sum(), (delta * delta).sum(),
                                       torch.tensor(float(delta.numel()), dtype=torch.float64, device=dev)])
                    parallel.all_reduce_sum(mom, group)
                    m1, m2, cnt_d = (float(x) for x in mom)
                    sigma_hat = float(np.sqrt(max(m2 - m1 * m1 / cnt_d, 0.0) / (cnt_d - 1))) if cnt_d > 1 else 0.0
                else:
                    sigma_hat = float(delta.std()) if delta.numel() > 1 else 0.0
            record = {"step": step, "energy": energy, "mc_error": err, "acceptance": acceptance,
                      "sigma_hat": sigma_hat, "bound_pinsker": pinsker_tv_bound(sigma_hat),
                      "bound_theorem3": theorem3_gaussian_bound(sigma_hat, 0.0, 0.0), "kappa": update.kappa}
            if config.sr_solver == "cg":
                record["cg_iterations"] = update.iterations
            if config.track_timings:
                torch.cuda.synchronize(dev)
                record["sampling_seconds"] = t_update - t_sample
                record["update_seconds"] = time.perf_counter() - t_update
            if config.reference_energy is not None:
                record["rel_error"] = abs(energy - config.reference_energy) / abs(config.reference_energy)
            records.append(record)
        params = new_params
    return TrainResult(records, params, force_history)
