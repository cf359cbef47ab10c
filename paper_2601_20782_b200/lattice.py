"""Lattices and bond lists (mirror of the reference lattice.py:118-182).

Spin convention s_i = 1 - 2*bit_i; 2D sites row-major (r, c) -> r*L + c; bonds
are (i<j) pairs, sorted, deduplicated — identical to LatticeSpec.bonds so the
device Hamiltonian kernels see the same bond order as the reference.  Unlike
the reference's SpinConfiguration (N <= 62), device configurations are packed
uint32 words, so any N up to MAX_DEVICE_SITES works.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

ENUMERATION_LIMIT = 14
MAX_DEVICE_SITES = 1024


@dataclass(frozen=True)
class LatticeSpec:
    shape: tuple
    periodic: bool
    bonds: tuple = field(init=False)

    def __post_init__(self):
        if len(self.shape) == 1:
            (n,) = self.shape
            if n < 1:
                raise ValueError("chain length must be >= 1")
            if self.periodic and n < 3:
                raise ValueError("periodic chain requires n >= 3")
            bonds = [(i, i + 1) for i in range(n - 1)]
            if self.periodic:
                bonds.append((0, n - 1))
        elif len(self.shape) == 2:
            rows, cols = self.shape
            if rows != cols:
                raise ValueError("only square 2D lattices are supported")
            length = rows
            if self.periodic and length < 3:
                raise ValueError("periodic square lattice requires L >= 3")
            if length < 2:
                raise ValueError("square lattice requires L >= 2")
            bonds = []
            for r in range(length):
                for c in range(length):
                    site = r * length + c
                    right = site + 1 if c + 1 < length else (r * length if self.periodic else None)
                    down = site + length if r + 1 < length else (c if self.periodic else None)
                    for other in (right, down):
                        if other is not None:
                            bonds.append((min(site, other), max(site, other)))
        else:
            raise ValueError("shape must be (n,) or (L, L)")
        object.__setattr__(self, "bonds", tuple(sorted(set(bonds))))

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
        """Next-nearest-neighbour (i<j) pairs, sorted, deduplicated, excluding
        nearest-neighbour pairs (beyond the reference: J1-J2 models).  Chain:
        (i, i+2); square: both diagonals; periodic wrap as for `bonds`."""
        pairs = set()
        if len(self.shape) == 1:
            (n,) = self.shape
            for i in range(n):
                j = i + 2
                if j >= n:
                    if not self.periodic:
                        continue
                    j -= n
                if i != j:
                    pairs.add((min(i, j), max(i, j)))
        else:
            length = self.shape[0]
            for r in range(length):
                for c in range(length):
                    for dc in (1, -1):
                        rr, cc = r + 1, c + dc
                        if not (0 <= cc < length and rr < length):
                            if not self.periodic:
                                continue
                            rr, cc = rr % length, cc % length
                        a, b = r * length + c, rr * length + cc
                        if a != b:
                            pairs.add((min(a, b), max(a, b)))
        pairs -= set(self.bonds)
        return np.array(sorted(pairs), dtype=np.int64).reshape(-1, 2)

    def sublattice(self) -> np.ndarray:
        """Checkerboard sublattice index (0/1) of every site; raises if the
        nearest-neighbour bonds do not join the two sublattices (Marshall sign
        needs a bipartite lattice: open, or periodic with even length)."""
        if len(self.shape) == 1:
            sub = np.arange(self.shape[0]) % 2
        else:
            length = self.shape[0]
            r, c = np.divmod(np.arange(length * length), length)
            sub = (r + c) % 2
        bonds = self.bond_array()
        if bonds.size and np.any(sub[bonds[:, 0]] == sub[bonds[:, 1]]):
            raise ValueError("lattice is not bipartite (periodic with odd length)")
        return sub.astype(np.int64)


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
