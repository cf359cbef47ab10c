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
    st = host[-1:].view(torch.int64).numpy()[0]
    if st[0] != 0:
        bad = int(st[1])
        raise EvaluationFailureError("non-finite local energy", context={"bits": bits[bad].copy()})
    # the (re, im) pairs are complex128 already: a zero-copy view of the pinned block
    return host[:-1].numpy().view(np.complex128)[:, 0]


def _moments_out(x, fn, *args):
    import torch

    partials = torch.empty(int(nat.load().mpv_cg_partials_len()), dtype=torch.float64, device=x.device)
    out = torch.empty(3, dtype=torch.float64, device=x.device)
    nat.call(fn, *args, partials.data_ptr(), out.data_ptr(), nat.stream_handle(x.device))
    return [float(v) for v in out.cpu()]


def device_mc_error(eps_u, inverse, n_samples: int, n_chains: int) -> float:
    """Split-chain MC error (vmc.py:592-604 with mc_error, vmc.py:311-317) on the
    device: per-chain means of Re eps over the chain-major sample rows (sample
    row -> unique row through `inverse`), then sqrt(var(means, ddof=1) / C) from
    two-pass moments (mpv_chain_stats).  One chain: the samples themselves."""
    import torch

    eps_ri = torch.view_as_real(eps_u.contiguous()).contiguous() if eps_u.is_complex() else eps_u
    inverse = inverse.to(torch.int64).contiguous()
    C = n_chains if n_chains > 1 else int(n_samples)
    base, extra = divmod(int(n_samples), C)
    means = torch.empty(C, dtype=torch.float64, device=eps_u.device)
    _, ss, c = _moments_out(eps_u, "mpv_chain_stats", eps_ri.data_ptr(), inverse.data_ptr(), C, 0, base, extra, 0,
                            means.data_ptr())
    if c < 2:
        raise DegenerateInputError("need >= 2 values")
    return float(np.sqrt(ss / (c - 1) / c))


def device_std(x) -> float:
    """Unbiased standard deviation of a real device vector (two-pass, mpv_moments)."""
    x = x.contiguous()
    _, ss, n = _moments_out(x, "mpv_moments", x.data_ptr(), x.numel())
    return float(np.sqrt(ss / (n - 1)))


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


def _params_flat(params, dev):
    """[a | b | W row-major] complex on the device (RbmParameters.flatten order)."""
    import torch

    return torch.from_numpy(np.ascontiguousarray(params.flatten())).to(dev)


def grad_log_psi_device(params, bits_u8, device=None):
    """O(x) = d log psi / d theta (rbm.py:307-325) for a (U, N) uint8 device
    tensor: columns a, b, W row-major; complex128 [U, P] on the device
    (mpv_logderiv_tanh for tanh(b + W x), mpv_logderiv_dense for the layout)."""
    import torch

    dev = bits_u8.device
    U, N = bits_u8.shape
    packed = torch.empty((U, (N + 31) // 32), dtype=torch.int32, device=dev)
    if U:
        nat.call("mpv_pack_bits", bits_u8.data_ptr(), U, N, packed.data_ptr(), nat.stream_handle(dev))
    fo = FactoredLogDerivatives(params, packed)
    return fo.dense()


def forces(*, o, eps, weights=None):
    """F_k = E[conj(O_k) eps] - E[conj(O_k)] E[eps] (vmc.py:145-165), device tensors
    (elementwise products and column sums; no BLAS)."""
    if o.shape[0] != eps.numel() or eps.numel() == 0:
        raise DegenerateInputError("need at least one (O, eps) pair")
    if weights is None:
        if eps.numel() < 2:
            raise DegenerateInputError("need >= 2 samples")
        w = eps.new_full((eps.numel(),), 1.0 / eps.numel()).real
    else:
        w = weights.to(eps.real.dtype)
    oc = o.conj()
    we = w.to(eps.dtype) * eps
    return (oc * we[:, None]).sum(dim=0) - (oc * w.to(eps.dtype)[:, None]).sum(dim=0) * we.sum()


def s_matrix(*, o, weights=None):
    """S = E[conj(O) O^T] - E[conj O] E[O^T], Hermitised (vmc.py:168-188): the
    centred O and mpv_sr_smatrix (a tiled f64 kernel, Hermitian by construction)."""
    import torch

    if o.shape[0] == 0:
        raise DegenerateInputError("empty sample set")
    U, P = o.shape
    w = (torch.full((U,), 1.0 / U, dtype=torch.float64, device=o.device) if weights is None
         else weights.to(torch.float64).contiguous())
    mean = (o * w.to(o.dtype)[:, None]).sum(dim=0)
    c = (o - mean[None, :]).contiguous()
    s = torch.empty((P, P), dtype=torch.complex128, device=o.device)
    nat.call("mpv_sr_smatrix", c.data_ptr(), w.data_ptr(), U, P, s.data_ptr(), nat.stream_handle(o.device))
    return s


def s_matrix_centred(c, weights):
    """sum_s w_s conj(C_s) C_s^T for an already centred dense C (mpv_sr_smatrix)."""
    import torch

    U, P = c.shape
    w = weights.to(torch.float64).contiguous()
    s = torch.empty((P, P), dtype=torch.complex128, device=c.device)
    nat.call("mpv_sr_smatrix", c.contiguous().data_ptr(), w.data_ptr(), U, P, s.data_ptr(), nat.stream_handle(c.device))
    return s


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
    and S 6.6 GB).  T comes from mpv_logderiv_tanh (DMMA GEMM over the bits,
    complex tanh epilogue); O v and O^H u run in csrc/logderiv.cuh as DMMA GEMMs
    over the bits with fused epilogues (weights and sum_s u_s fused).
    `reduce` (optional) all-reduces sums over samples across ranks."""

    def __init__(self, params, packed, reduce=None, bits_u8=None):
        import torch

        dev = packed.device
        if packed.dtype == torch.uint8:  # (U, N) 0/1 rows: pack them on the device
            bits_u8 = packed
            U, N = packed.shape
            packed = torch.empty((U, (N + 31) // 32), dtype=torch.int32, device=dev)
            if U:
                nat.call("mpv_pack_bits", bits_u8.contiguous().data_ptr(), U, N, packed.data_ptr(),
                         nat.stream_handle(dev))
        self.N, self.M = params.n_visible, params.n_hidden
        self.P = self.N + self.M + self.M * self.N
        self.packed = packed.contiguous()
        self.U = self.packed.shape[0]
        self.packed_u8 = bits_u8
        self.device = dev
        self.scratch = torch.empty(nat.load().mpv_logderiv_scratch_bytes(self.U, self.N, self.M), dtype=torch.uint8,
                                   device=dev)
        self.t = torch.empty((self.U, self.M), dtype=torch.complex128, device=dev)
        nat.call("mpv_logderiv_tanh", _params_flat(params, dev).data_ptr(), self.packed.data_ptr(), self.U, self.N,
                 self.M, self.t.data_ptr(), self.scratch.data_ptr(), nat.stream_handle(dev))
        self.reduce = reduce or (lambda z: z)
        self.reduce_is_local = reduce is None

    def _s(self):
        return nat.stream_handle(self.device)

    def o_v(self, v, w=None):
        """q_s = w_s (O v)_s (w None: 1)."""
        import torch

        v = v.resolve_conj().contiguous()
        q = torch.empty(self.U, dtype=torch.complex128, device=self.device)
        nat.call("mpv_logderiv_ov", self.t.data_ptr(), self.packed.data_ptr(), self.U, self.N, self.M, v.data_ptr(),
                 w.data_ptr() if w is not None else None, q.data_ptr(), self.scratch.data_ptr(), self._s())
        return q

    def oh_u(self, u, w=None, with_sum=False):
        """sum_s conj(O_s) w_s u_s (local sums; callers reduce); with_sum: also
        sum_s w_s u_s, returned as element P of a P+1 vector."""
        import torch

        u = u.resolve_conj().contiguous()
        out = torch.empty(self.P + 1, dtype=torch.complex128, device=self.device)
        nat.call("mpv_logderiv_ohu", self.t.data_ptr(), self.packed.data_ptr(), self.U, self.N, self.M, u.data_ptr(),
                 w.data_ptr() if w is not None else None, out.data_ptr(),
                 out[self.P:].data_ptr() if with_sum else None, self.scratch.data_ptr(), self._s())
        return out if with_sum else out[:self.P]

    def dense(self, obar=None):
        """O_s - obar as a dense complex [U, P] tensor (small P only)."""
        import torch

        o = torch.empty((self.U, self.P), dtype=torch.complex128, device=self.device)
        nat.call("mpv_logderiv_dense", self.t.data_ptr(), self.packed.data_ptr(), self.U, self.N, self.M,
                 obar.resolve_conj().contiguous().data_ptr() if obar is not None else None, o.data_ptr(),
                 self._s())
        return o

    def statistics(self, eps, weights):
        """(F, energy, obar) of the reference estimators (vmc.py:145-165) with one
        reduction across ranks: F = sum_w conj(O) eps - (sum_w conj O)(sum_w eps),
        obar = sum_w O."""
        import torch

        w = weights.to(torch.float64).contiguous()
        ones = torch.ones(self.U, dtype=torch.complex128, device=self.device)
        first = torch.cat([self.oh_u(eps, w, with_sum=True), self.oh_u(ones, w)])
        first = self.reduce(first)
        P = self.P
        s_oe, e, s_o = first[:P], first[P], first[P + 1:]
        return s_oe - s_o * e, e, s_o.conj().resolve_conj()


def sr_step_cg(o: FactoredLogDerivatives, eps, weights, lambda_shift: float, eta: float,
               tol: float = 1e-10, maxiter: int = 1000, batch: int = 16):
    """SR update without forming S (matrix-free conjugate gradients on the
    Hermitian positive-definite S + lambda I; beyond the reference's dense
    Cholesky, vmc.py:202-229, which does not fit config 2).  Same estimators:
    F = sum_w conj(O) eps - (sum_w conj O)(sum_w eps),
    S v = sum_w conj(O) (O v) - conj(Obar)(Obar v).

    Device-resident (csrc/sr.cuh): the CG scalars and the convergence flag stay
    on the device, a converged solve turns the remaining iterations of a batch
    into no-ops, and the host reads the flag once per `batch` iterations
    (single process: mpv_cg_run; across ranks: one all-reduce of O^H(w O p)
    per iteration between mpv_cg_apply and mpv_cg_step).
    Returns (SrUpdate, F, energy)."""
    import torch

    if lambda_shift < 0:
        raise ValueError("lambda must be >= 0")
    if eta <= 0:
        raise ValueError("eta must be > 0")
    w = weights.to(torch.float64).contiguous()
    f, e, obar = o.statistics(eps, w)
    f = f.resolve_conj().contiguous()
    obar = obar.resolve_conj().contiguous()
    dev, P = o.device, o.P
    c128 = lambda n: torch.empty(n, dtype=torch.complex128, device=dev)  # noqa: E731
    g, r, pv, ap, q = c128(P), c128(P), c128(P), c128(P), c128(max(o.U, 1))
    yy = c128(P + 1)
    partials = torch.empty(int(nat.load().mpv_cg_partials_len()), dtype=torch.float64, device=dev)
    scalars = torch.zeros(8, dtype=torch.float64, device=dev)
    cg = nat.CG(o.N, o.M, o.U, o.t.data_ptr(), o.packed.data_ptr(), w.data_ptr(), obar.data_ptr(),
                float(lambda_shift), g.data_ptr(), r.data_ptr(), pv.data_ptr(), ap.data_ptr(), yy.data_ptr(),
                yy[P:].data_ptr(), q.data_ptr(), partials.data_ptr(), scalars.data_ptr(), o.scratch.data_ptr(),
                o.scratch.numel())
    cgp = ctypes.byref(cg)
    st = nat.stream_handle(dev)
    nat.call("mpv_cg_init", cgp, f.data_ptr(), float(tol), int(maxiter), st)
    host = torch.empty(8, dtype=torch.float64, pin_memory=True)
    while True:
        if o.reduce_is_local:
            nat.call("mpv_cg_run", cgp, int(batch), st)
        else:
            for _ in range(batch):
                nat.call("mpv_cg_apply", cgp, pv.data_ptr(), yy.data_ptr(), yy[P:].data_ptr(), st)
                o.reduce(yy)
                nat.call("mpv_cg_step", cgp, st)
        host.copy_(scalars, non_blocking=True)
        torch.cuda.current_stream(dev).synchronize()
        if host[3] != 0.0:
            break
    it = int(host[2])
    fn = float(torch.linalg.vector_norm(f))
    # residual of the returned g with one more application of S + lambda
    nat.call("mpv_cg_apply", cgp, g.data_ptr(), yy.data_ptr(), yy[P:].data_ptr(), st)
    o.reduce(yy)
    nat.call("mpv_cg_apply_finish", cgp, g.data_ptr(), yy.data_ptr(), yy[P:].data_ptr(), ap.data_ptr(), st)
    residual = float(torch.linalg.vector_norm(ap - f)) / fn if fn > 0 else 0.0
    if fn > 0 and residual > max(10 * tol, 1e-9):
        raise SolverError(f"SR conjugate-gradient residual {residual:.3e} after {it} iterations")
    return SrUpdate(g, float("nan"), residual, lambda_shift, eta, it), f, float(e.real)


def _gather_rows(x, group=None):
    """Concatenate a per-rank tensor along dim 0 over all ranks (rank order);
    returns (all rows, this rank's first row).  Ranks may hold different counts."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    n = torch.tensor([x.shape[0]], dtype=torch.int64, device=x.device)
    counts = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(counts, n, group=group)
    counts = [int(c) for c in counts]
    nmax = max(counts)
    pad = torch.zeros((nmax,) + tuple(x.shape[1:]), dtype=x.dtype, device=x.device)
    pad[:x.shape[0]] = x
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    rank = dist.get_rank(group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)]), sum(counts[:rank])


def sr_step_minsr(o: FactoredLogDerivatives, eps, weights, lambda_shift: float, eta: float,
                  precision: str = "f64", group=None):
    """The same SR update solved in sample space (minSR; beyond the reference).

    With O~ = W^{1/2} (O - 1 obar^T) the reference's estimators are S = O~^H O~
    and F = O~^H e~ (e~ = W^{1/2} (eps - ebar)), and the push-through identity
    gives g = (S + lambda)^-1 F = O~^H (O~ O~^H + lambda)^-1 e~ exactly: a U x U
    Cholesky instead of a P x P one (cheaper whenever U < P).  The Gram matrix
    never needs O: mpv_minsr_gram forms it from the factors (common set bits of
    the packed rows, T T^H) with the centring and weights fused, in f64 or
    (precision="f32", the north star's "minSR in f32") f32 with an f32 solve.
    Across ranks (o.reduce set, `group`): the factors are all-gathered, every rank
    builds its own block of rows of the U x U matrix, the rows are all-gathered,
    every rank solves the same system, and O^H y sums per rank then all-reduces."""
    import torch

    if lambda_shift < 0:
        raise ValueError("lambda must be >= 0")
    if eta <= 0:
        raise ValueError("eta must be > 0")
    if precision not in ("f64", "f32"):
        raise ValueError("precision must be 'f64' or 'f32'")
    w = weights.to(torch.float64).contiguous()
    f, e, obar = o.statistics(eps, w)
    d = o.o_v(obar.conj())  # d_s = (O conj(obar))_s
    sw = torch.sqrt(w)
    et = (sw.to(torch.complex128) * (eps - e)).contiguous()
    sharded = not o.reduce_is_local
    if sharded:
        t_all, row0 = _gather_rows(o.t, group)
        bits_all, _ = _gather_rows(o.packed, group)
        d_all, _ = _gather_rows(d, group)
        w_all, _ = _gather_rows(w, group)
        et_all, _ = _gather_rows(et, group)
    else:
        t_all, bits_all, d_all, w_all, et_all, row0 = o.t, o.packed, d, w, et, 0
    U_all = t_all.shape[0]
    ctype = torch.complex64 if precision == "f32" else torch.complex128
    rows = torch.empty((o.U, U_all), dtype=ctype, device=o.device)
    obar2 = float(torch.vdot(obar, obar).real)
    nat.call("mpv_minsr_gram", o.t.data_ptr(), o.packed.data_ptr(), o.U, row0, t_all.contiguous().data_ptr(),
             bits_all.contiguous().data_ptr(), U_all, o.N, o.M, d_all.contiguous().data_ptr(),
             w_all.contiguous().data_ptr(), obar2, float(lambda_shift), 1 if precision == "f32" else 0,
             rows.data_ptr(), nat.stream_handle(o.device))
    k = _gather_rows(rows, group)[0] if sharded else rows
    k = 0.5 * (k + k.mH)
    rhs = et_all.to(ctype)
    L, info = torch.linalg.cholesky_ex(k)
    if int(info) != 0:
        raise SolverError("sample-space matrix O~ O~^H + lambda I is not positive definite")
    y = torch.cholesky_solve(rhs[:, None], L)[:, 0]
    y = y + torch.cholesky_solve((rhs - k @ y)[:, None], L)[:, 0]  # one refinement pass
    residual = float(torch.linalg.norm(k @ y - rhs) / max(float(torch.linalg.norm(rhs)), 1e-300))
    z = (sw.to(torch.complex128) * y[row0:row0 + o.U].to(torch.complex128)).contiguous()
    gz = o.reduce(o.oh_u(z, with_sum=True))
    g = gz[:o.P] - obar.conj() * gz[o.P]
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
    minsr_precision: str = "f64"  # "f64" or "f32" (Gram matrix and solve)

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
        red = (lambda z: parallel.all_reduce_sum(z, group)) if world > 1 else None
        fo = FactoredLogDerivatives(params, uniq, red)
        if config.sr_solver == "cg":
            update, f, energy = sr_step_cg(fo, eps, est_w, config.lambda_shift, config.eta, config.cg_tol,
                                           config.cg_maxiter)
        elif config.sr_solver == "minsr":
            update, f, energy = sr_step_minsr(fo, eps, est_w, config.lambda_shift, config.eta,
                                              config.minsr_precision, group)
        else:
            # the reference's dense path: F and obar from the factored kernels, the
            # centred dense O, S = sum_w conj(C) C^T (mpv_sr_smatrix), Cholesky
            f, e_glob, obar = fo.statistics(eps, est_w)
            s = s_matrix_centred(fo.dense(obar), est_w)
            if world > 1:
                parallel.all_reduce_sum(s, group)
            energy = float(e_glob.real)
            update = sr_step(f, s, config.lambda_shift, config.eta, config.compute_kappa)
        theta = params.flatten() - config.eta * update.g.cpu().numpy()
        nvtx.range_pop()
        new_params = rbm.RbmParameters.from_flat(theta, params.n_visible, params.n_hidden)
        if exact_mode:
            err = 0.0
        elif world > 1:
            err = parallel.energy_statistics(eps.real[inverse], counts, 0, 1, group)["mc_error"]
        else:
            err = device_mc_error(eps, inverse, config.n_samples, n_chains)
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
                    sigma_hat = device_std(delta) if delta.numel() > 1 else 0.0
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
