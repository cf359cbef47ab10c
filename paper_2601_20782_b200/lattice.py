"""Lattices and bond lists.  API names follow the reference (`lattice.py:118-182`:
LatticeSpec(shape, periodic), .chain, .square, n_sites, bonds, bond_array);
the construction is this package's own: bonds are generated from lattice
displacement vectors over site coordinates, so nearest and next-nearest
neighbours share one code path.

Conventions (they fix the device kernels' bond order): spin s = 1 - 2 bit;
2D sites row-major, site(r, c) = r L + c; a bond is an (i < j) pair; the list
is sorted and free of duplicates (small periodic lattices wrap onto the same
pair).  Device configurations are packed uint32 words (any N up to
MAX_DEVICE_SITES), unlike the reference's 62-site integer codes.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ENUMERATION_LIMIT = 14
MAX_DEVICE_SITES = 1024


def _pairs(coords: np.ndarray, extent: int, periodic: bool, disp) -> set:
    """(i < j) pairs joining every site to site + disp (coordinates in [0, extent))."""
    target = coords + np.asarray(disp)[None, :]
    if periodic:
        target %= extent
        keep = np.ones(len(coords), dtype=bool)
    else:
        keep = np.all((target >= 0) & (target < extent), axis=1)
    dims = coords.shape[1]
    weights = extent ** np.arange(dims - 1, -1, -1)  # row-major site index
    a = coords[keep] @ weights
    b = target[keep] @ weights
    return {(int(min(x, y)), int(max(x, y))) for x, y in zip(a, b) if x != y}


@dataclass(frozen=True)
class LatticeSpec:
    shape: tuple
    periodic: bool
    bonds: tuple = field(init=False)

    def __post_init__(self):
        dims = len(self.shape)
        if dims not in (1, 2):
            raise ValueError(f"lattice shape must be (n,) or (L, L), got {self.shape}")
        if dims == 2 and self.shape[0] != self.shape[1]:
            raise ValueError(f"2D lattices are square here, got {self.shape}")
        extent = int(self.shape[0])
        smallest = 1 if dims == 1 else 2
        if extent < smallest or (self.periodic and extent < 3):
            raise ValueError(f"lattice {self.shape} is too small ({'periodic needs >= 3' if self.periodic else ''})")
        nn = set()
        for axis in range(dims):
            disp = np.zeros(dims, dtype=np.int64)
            disp[axis] = 1
            nn |= _pairs(self._coords(), extent, self.periodic, disp)
        object.__setattr__(self, "bonds", tuple(sorted(nn)))

    def _coords(self) -> np.ndarray:
        extent = int(self.shape[0])
        if len(self.shape) == 1:
            return np.arange(extent)[:, None]
        r, c = np.divmod(np.arange(extent * extent), extent)
        return np.stack([r, c], axis=1)

    @classmethod
    def chain(cls, n: int, periodic: bool = False) -> "LatticeSpec":
        return cls((n,), periodic)

    @classmethod
    def square(cls, length: int, periodic: bool = True) -> "LatticeSpec":
        return cls((length, length), periodic)

    @property
    def n_sites(self) -> int:
        return int(np.prod(self.shape))

    @property
    def boundary(self) -> str:
        return "periodic" if self.periodic else "open"

    def bond_array(self) -> np.ndarray:
        return np.array(self.bonds, dtype=np.int64).reshape(-1, 2)

    def next_nearest_bonds(self) -> np.ndarray:
        """Next-nearest-neighbour (i < j) pairs (beyond the reference: J1-J2
        models): chain (i, i+2), square lattice both diagonals; same wrap rule
        as the bonds, pairs that are also nearest neighbours excluded."""
        extent = int(self.shape[0])
        disps = [(2,)] if len(self.shape) == 1 else [(1, 1), (1, -1)]
        pairs = set()
        for d in disps:
            pairs |= _pairs(self._coords(), extent, self.periodic, d)
        pairs -= set(self.bonds)
        return np.array(sorted(pairs), dtype=np.int64).reshape(-1, 2)

    def sublattice(self) -> np.ndarray:
        """Checkerboard sublattice (0/1) of every site; a lattice whose bonds join
        equal sublattices (periodic, odd length) is rejected - the Marshall sign
        needs a bipartite lattice."""
        parity = self._coords().sum(axis=1) % 2
        bonds = self.bond_array()
        if bonds.size and np.any(parity[bonds[:, 0]] == parity[bonds[:, 1]]):
            raise ValueError(f"{self.shape} {self.boundary} lattice is not bipartite")
        return parity.astype(np.int64)


def enumerate_bits(n: int) -> np.ndarray:
    """(2^n, n) bit matrix in ascending code order (lattice.py:95-101)."""
    if not 1 <= n <= ENUMERATION_LIMIT:
        from .errors import EnumerationTooLargeError

        raise EnumerationTooLargeError(f"enumeration supports 1 <= n <= {ENUMERATION_LIMIT}, got {n}")
    codes = np.arange(1 << n, dtype=np.uint64)
    return ((codes[:, None] >> np.arange(n, dtype=np.uint64)[None, :]) & 1).astype(np.uint8)


def pack_bits(bits) -> np.ndarray:
    """uint8 (B, N) -> uint32 (B, ceil(N/32)) words, bit k of a row in word k>>5, bit k&31."""
    bits = np.ascontiguousarray(np.atleast_2d(bits), dtype=np.uint8)
    b, n = bits.shape
    words = (n + 31) // 32
    padded = np.zeros((b, words * 32), dtype=np.uint8)
    padded[:, :n] = bits
    packed = np.packbits(padded.reshape(b, words, 4, 8)[..., ::-1], axis=-1)[..., 0]
    return np.ascontiguousarray(packed).view(np.uint32).reshape(b, words) if b else np.zeros((0, words), np.uint32)


def unpack_bits(words, n: int) -> np.ndarray:
    words = np.ascontiguousarray(np.atleast_2d(words), dtype=np.uint32)
    b = words.shape[0]
    bytes_ = words.view(np.uint8).reshape(b, -1)
    bits = np.unpackbits(bytes_, axis=1, bitorder="little")
    return np.ascontiguousarray(bits[:, :n])
