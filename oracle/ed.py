"""Dense exact diagonalisation — test infrastructure only.

Restates the reference's ``hamiltonians.dense_matrix`` / ``exact_ground_state``
(/root/reference/pkg/src/mpvmc/hamiltonians.py:95-150): the 2^n x 2^n real
symmetric Hamiltonian in configuration-code order (spin s = 1 - 2 bit),
TFIM  H = J sum_bonds s_i s_j + h sum_i sigma^x_i,
Heisenberg  H = J sum_bonds s_i s_j + 2J (swap of anti-aligned bond spins).
Pinned to the reference's own E0 values (tests/golden/ed.npz).
"""
from __future__ import annotations

import numpy as np


def dense_matrix(kind, n, bonds, j, h=0.0):
    dim = 1 << n
    codes = np.arange(dim)
    bits = (codes[:, None] >> np.arange(n)) & 1
    spins = 1 - 2 * bits
    bonds = np.asarray(bonds, dtype=np.int64).reshape(-1, 2)
    diag = (spins[:, bonds[:, 0]] * spins[:, bonds[:, 1]]).sum(axis=1).astype(np.float64) if bonds.size else \
        np.zeros(dim)
    mat = np.zeros((dim, dim))
    mat[codes, codes] = j * diag
    if kind == "tfim":
        for i in range(n):
            mat[codes, codes ^ (1 << i)] += h
    else:
        for i, k in bonds:
            differ = bits[:, i] != bits[:, k]
            mat[codes[differ], codes[differ] ^ ((1 << int(i)) | (1 << int(k)))] += 2.0 * j
    return mat


def ground_energy(kind, n, bonds, j, h=0.0):
    return float(np.linalg.eigvalsh(dense_matrix(kind, n, bonds, j, h))[0])


def sparse_matrix(terms, n):
    """Sum of terms (kind, bonds, j, h) as a scipy CSR matrix (n up to ~20)."""
    import scipy.sparse as sp

    dim = 1 << n
    codes = np.arange(dim)
    bits = ((codes[:, None] >> np.arange(n)) & 1).astype(np.int8)
    spins = (1 - 2 * bits).astype(np.int8)
    diag = np.zeros(dim)
    rows, cols, vals = [], [], []
    for kind, bonds, j, h in terms:
        bonds = np.asarray(bonds, dtype=np.int64).reshape(-1, 2)
        for i, k in bonds:
            diag += j * spins[:, i] * spins[:, k]
        if kind == "tfim":
            for i in range(n):
                rows.append(codes)
                cols.append(codes ^ (1 << i))
                vals.append(np.full(dim, float(h)))
        else:
            for i, k in bonds:
                differ = bits[:, i] != bits[:, k]
                rows.append(codes[differ])
                cols.append(codes[differ] ^ ((1 << int(i)) | (1 << int(k))))
                vals.append(np.full(int(differ.sum()), 2.0 * j))
    rows.append(codes)
    cols.append(codes)
    vals.append(diag)
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(dim, dim))


def ground_energy_sparse(terms, n):
    import scipy.sparse.linalg as sla

    return float(sla.eigsh(sparse_matrix(terms, n), k=1, which="SA")[0][0])
