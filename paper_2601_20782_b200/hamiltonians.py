"""TFIM and Heisenberg specs (mirror of the reference hamiltonians.py:28-46).

Conventions as in the reference (hamiltonians.py:1-7): TFIM
H = J sum_<ij> sz_i sz_j + h sum_i sx_i (both +); Heisenberg in Pauli matrices,
a bond contributes +-J on the diagonal and 2J off-diagonally when the spins
differ.  The device local-energy kernel (csrc/energy.cuh) uses them.

Beyond the reference (parity pinned by exact H|psi> on
enumerable lattices in tests/test_gpu_energy_models.py): `marshall=True` applies
the Marshall sign psi_M(x) = (-1)^{#up spins on sublattice A} psi(x) (it flips
the sign of every off-diagonal element on a bond joining the sublattices), and
`J1J2Spec` adds next-nearest-neighbour bonds with coupling j2.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .lattice import LatticeSpec


@dataclass(frozen=True)
class TfimSpec:
    lattice: LatticeSpec
    j: float
    h: float

    def __post_init__(self):
        if not (np.isfinite(self.j) and np.isfinite(self.h)):
            raise ValueError("couplings must be finite")


@dataclass(frozen=True)
class HeisenbergSpec:
    lattice: LatticeSpec
    j: float
    marshall: bool = False

    def __post_init__(self):
        if not np.isfinite(self.j):
            raise ValueError("coupling must be finite")
        if self.marshall:
            self.lattice.sublattice()  # validates bipartiteness

    def couplings(self):
        """(bonds int64[nb, 2], diagonal J per bond, off-diagonal coefficient per bond)."""
        bonds = self.lattice.bond_array()
        jb = np.full(bonds.shape[0], float(self.j))
        return bonds, jb, _offdiag(self.lattice, bonds, jb, self.marshall)


@dataclass(frozen=True)
class J1J2Spec:
    """Heisenberg J1-J2 model (Pauli matrices, as HeisenbergSpec): nearest-
    neighbour bonds with j1, next-nearest with j2; optional Marshall sign."""

    lattice: LatticeSpec
    j1: float
    j2: float
    marshall: bool = False

    def __post_init__(self):
        if not (np.isfinite(self.j1) and np.isfinite(self.j2)):
            raise ValueError("couplings must be finite")
        if self.marshall:
            self.lattice.sublattice()

    def couplings(self):
        nn, nnn = self.lattice.bond_array(), self.lattice.next_nearest_bonds()
        bonds = np.concatenate([nn, nnn]).reshape(-1, 2)
        jb = np.concatenate([np.full(nn.shape[0], float(self.j1)), np.full(nnn.shape[0], float(self.j2))])
        return bonds, jb, _offdiag(self.lattice, bonds, jb, self.marshall)


def _offdiag(lattice, bonds, jb, marshall):
    coef = 2.0 * jb
    if marshall and bonds.size:
        sub = lattice.sublattice()
        coef = np.where(sub[bonds[:, 0]] != sub[bonds[:, 1]], -coef, coef)
    return coef
