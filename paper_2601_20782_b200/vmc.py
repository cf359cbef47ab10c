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
from .hamiltonians import HeisenbergSpec, TfimSpec
from .lattice import pack_bits


class EnergyKernel:
    """Device parameters + cosh/sinh tables of one (params, Hamiltonian) pair."""

    def __init__(self, spec, params, device=None):
        import torch

        nat.require_cuda()
        if isinstance(spec, TfimSpec):
            self.ham, self.J, self.h = nat.HAM_TFIM, float(spec.j), float(spec.h)
        elif isinstance(spec, HeisenbergSpec):
            self.ham, self.J, self.h = nat.HAM_HEISENBERG, float(spec.j), 0.0
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
        bonds = spec.lattice.bond_array().astype(np.int32)
        self.n_bonds = bonds.shape[0]
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
        nat.call("mpv_local_energies", self.N, self.M, self.a.data_ptr(), self.b.data_ptr(), self.w_t.data_ptr(),
                 self.ham, self._bonds_ptr(), self.n_bonds, self.J, self.h, self.tables.data_ptr(),
                 packed_bits.data_ptr(), B, out.data_ptr(), status.data_ptr(), nat.stream_handle(self.device))
        return out, status


def _energy_kernel(spec, log_amplitude):
    from .rbm import LogPsiEvaluator

    if not isinstance(log_amplitude, LogPsiEvaluator):
        raise TypeError("local_energies needs a device evaluator from rbm.log_psi_evaluator "
                        f"(got {type(log_amplitude).__name__}; there is no host-callable fallback)")
    key = (type(spec).__name__, spec.lattice, float(spec.j), float(getattr(spec, "h", 0.0)))
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
    eps = out.cpu().numpy()
    st = status.cpu().numpy()
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
