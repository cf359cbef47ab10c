"""TFIM and Heisenberg specs (mirror of the reference hamiltonians.py:28-46).

Conventions as in the reference (hamiltonians.py:1-7): TFIM
H = J sum_<ij> sz_i sz_j + h sum_i sx_i (both +); Heisenberg in Pauli matrices,
a bond contributes +-J on the diagonal and 2J off-diagonally when the spins
differ.  The device local-energy kernel (csrc/local_energy.cu) uses them.
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

    def __post_init__(self):
        if not np.isfinite(self.j):
            raise ValueError("coupling must be finite")
